// gbs_acoustic2d_tma.cuh -- 2-D linear acoustics substep kernel fed by the
// Tensor Memory Accelerator (cp.async.bulk.tensor, SASS UTMALDG) through a
// D-stage full/empty mbarrier pipeline with a dedicated producer warp.
//
//   p_t = -(u_x + v_y),  u_t = -p_x,  v_t = -p_y     (BASELINE.json configs 2-3)
//
// One launch = one FE / LF / final substep of one GBS sequence (PAPER.md
// Eq. (1), lines 85-98), the FIN modes fused with the averaging and the
// weighted accumulate.  Same arithmetic, operand
// order and modes as gbs::acoustic2d_step (gbs_kernels.cuh), so the two agree
// bit for bit (tested); this one keeps D stages of loads in flight per SM
// independently of the register budget (the register-prefetch kernel holds one
// row ahead per thread and reached 0.78 of the copy bandwidth on C3).
//
// Tile: TX = 64 (x) by TY = 16 (y) points per iteration, 16 consumer warps
// (one row each, two consecutive x points per thread) + 1 producer warp; a CTA
// marches along y over ychunk rows, TY rows per iteration.  Per iteration the
// producer loads (boxes never cross the periodic boundary because the grid is
// a multiple of the tile; a wrapped halo box is a box at the wrapped coordinate):
//   p: centre column [TY + 2R][TX] (y stencil) + x strips [TY][R] (x stencil)
//   v: centre column [TY + 2R][TX] (y stencil)
//   u: centre [TY][TX] + x strips [TY][R] (x stencil)
//   previous level p, u, v and the accumulator (FINACC): [TY][TX] each
// Shared memory per stage: 7424 doubles (LF/FIN0), 10496 (FINACC), 4352 (FE).
#pragma once

#include "gbs_wave3d_tma.cuh"

namespace gbs {
namespace tma {

template <int R, int MODE>
struct AcLayout {
    static constexpr int COL = (TY + 2 * R) * TX;          // centre column with y halos
    static constexpr int STRIP = TY * R;
    static constexpr int PT = COL + 2 * STRIP;             // p tile
    static constexpr int VT = COL;                         // v column
    static constexpr int UT = TY * TX + 2 * STRIP;         // u row band
    static constexpr int PWT = TY * TX;
    static constexpr int NP = (MODE == MODE_FE) ? 0 : (MODE == MODE_FINACC ? 6 : 3);
    static constexpr int O_VT = PT, O_UT = PT + VT, O_PW = PT + VT + UT;
    static constexpr int STAGE = PT + VT + UT + NP * PWT;
    static constexpr int D = (MODE == MODE_FINACC) ? 2 : 3;
    static constexpr size_t stage_doubles = (size_t)D * STAGE;
    static constexpr size_t bytes = stage_doubles * 8 + (2 * D) * 8;
    static constexpr uint32_t stage_bytes = STAGE * 8;
    static_assert((COL * 8) % 128 == 0 && (STRIP * 8) % 128 == 0 && (PWT * 8) % 128 == 0,
                  "TMA destinations need 128 B alignment");
};

// Tensor maps of one launch: 3-D views [1][ny_alloc][nx] of each field buffer
// (ghost rows included in slab mode; y coordinate = y + ybase).
struct AcMaps {
    CUtensorMap s_a[3], s_b[3], s_c[3];   // current level p, u, v: TXxTY, TXxR, RxTY boxes
    CUtensorMap p[3];                     // previous level (TXxTY)
    CUtensorMap acc[3];                   // accumulator (TXxTY)
};

template <int R, int MODE, bool SLAB>
__global__ void __launch_bounds__(544, 1)
acoustic2d_step_tma(const __grid_constant__ AcMaps M, const Acoustic2DArgs A, const int ybase) {
    using L = AcLayout<R, MODE>;
    constexpr int D = L::D, STAGE = L::STAGE, PWT = L::PWT;
    extern __shared__ __align__(128) double smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::stage_doubles);
    uint64_t* empty = full + D;

    const int tx = threadIdx.x, ty = threadIdx.y, lane = tx;
    const int nx = A.nx, ny = A.ny;
    const int x0 = blockIdx.x * TX;
    const int ys = A.ylo + blockIdx.y * A.ychunk + (blockIdx.y ? A.yskip : 0);
    const int niter = (min(A.ychunk, A.yhi - ys) + TY - 1) / TY;   // ylo, ychunk, yhi: multiples of TY
    auto yc = [&](int y) -> int {              // tensor y coordinate of logical row y
        if constexpr (SLAB) return y + ybase;
        else return wrap_any(y, ny) + ybase;    // ybase: ghost rows of the layout (0 on plain grids)
    };

    if (ty == 0 && lane == 0) {
        for (int s = 0; s < D; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], TY); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (ty == TY) {
        // ===================== producer warp =====================
        if (lane != 0) return;
        for (int f = 0; f < 3; ++f) { prefetch_map(&M.s_a[f]); prefetch_map(&M.s_b[f]); prefetch_map(&M.s_c[f]); }
        const int xl = wrap_any(x0 - R, nx), xr = wrap_any(x0 + TX, nx);
        for (int i = 0; i < niter; ++i) {
            const int s = i % D;
            if (i >= D) mbar_wait(&empty[s], (uint32_t)(((i / D) - 1) & 1));
            mbar_expect_tx(&full[s], L::stage_bytes);
            double* st = smem + (size_t)s * STAGE;
            const int y = ys + i * TY;
            const int yt = yc(y - R), ym = yc(y), yb = yc(y + TY);
            // p: y halos + centre + x strips
            tma_load_3d(st, &M.s_b[0], x0, yt, 0, &full[s]);
            tma_load_3d(st + R * TX, &M.s_a[0], x0, ym, 0, &full[s]);
            tma_load_3d(st + (R + TY) * TX, &M.s_b[0], x0, yb, 0, &full[s]);
            tma_load_3d(st + L::COL, &M.s_c[0], xl, ym, 0, &full[s]);
            tma_load_3d(st + L::COL + L::STRIP, &M.s_c[0], xr, ym, 0, &full[s]);
            // v: y halos + centre
            double* v = st + L::O_VT;
            tma_load_3d(v, &M.s_b[2], x0, yt, 0, &full[s]);
            tma_load_3d(v + R * TX, &M.s_a[2], x0, ym, 0, &full[s]);
            tma_load_3d(v + (R + TY) * TX, &M.s_b[2], x0, yb, 0, &full[s]);
            // u: centre + x strips
            double* u = st + L::O_UT;
            tma_load_3d(u, &M.s_a[1], x0, ym, 0, &full[s]);
            tma_load_3d(u + PWT, &M.s_c[1], xl, ym, 0, &full[s]);
            tma_load_3d(u + PWT + L::STRIP, &M.s_c[1], xr, ym, 0, &full[s]);
            if constexpr (MODE != MODE_FE)
                for (int f = 0; f < 3; ++f) tma_load_3d(st + L::O_PW + f * PWT, &M.p[f], x0, ym, 0, &full[s]);
            if constexpr (MODE == MODE_FINACC)
                for (int f = 0; f < 3; ++f) tma_load_3d(st + L::O_PW + (3 + f) * PWT, &M.acc[f], x0, ym, 0, &full[s]);
        }
        return;
    }

    // ===================== consumer warps =====================
    // x-window sources of the thread's row: columns 2tx - R + 2k, from a tile whose
    // centre rows start at `crow` (row stride TX) and whose strips start at `strip`
    int xoff[R + 1];
#pragma unroll
    for (int k = 0; k <= R; ++k) {
        const int col = 2 * tx - R + 2 * k;
        xoff[k] = col < 0 ? -1 - (ty * R + (col + R))          // left strip (encoded negative)
                : col >= TX ? -1 - (L::STRIP + ty * R + (col - TX))
                            : ty * TX + col;
    }
    auto xwin = [&](const double* centre, const double* strips, double* w) {
#pragma unroll
        for (int k = 0; k <= R; ++k) {
            const double* src = xoff[k] >= 0 ? centre + xoff[k] : strips + (-1 - xoff[k]);
            const double2 t = *reinterpret_cast<const double2*>(src);
            w[2 * k] = t.x; w[2 * k + 1] = t.y;
        }
    };
    const int own = ty * TX + 2 * tx;                  // own column in a [TY][TX] box
    bool bad = false;
    for (int i = 0; i < niter; ++i) {
        const int s = i % D;
        mbar_wait(&full[s], (uint32_t)((i / D) & 1));
        const double* st = smem + (size_t)s * STAGE;
        const double* pc = st + R * TX;                // p centre rows (row 0 = tile row 0)
        const double* vc = st + L::O_VT + R * TX;
        double wu[2 * R + 2], wp[2 * R + 2];
        xwin(st + L::O_UT, st + L::O_UT + PWT, wu);
        xwin(pc, st + L::COL, wp);
        double dxu[2] = {0.0, 0.0}, dxp[2] = {0.0, 0.0}, dyv[2] = {0.0, 0.0}, dyp[2] = {0.0, 0.0};
        double2 vcen = *reinterpret_cast<const double2*>(vc + own);
#pragma unroll
        for (int j = 1; j <= R; ++j) {
            const double2 pu = *reinterpret_cast<const double2*>(pc + own + j * TX);
            const double2 pd = *reinterpret_cast<const double2*>(pc + own - j * TX);
            const double2 vu = *reinterpret_cast<const double2*>(vc + own + j * TX);
            const double2 vd = *reinterpret_cast<const double2*>(vc + own - j * TX);
            const double pup[2] = {pu.x, pu.y}, pdn[2] = {pd.x, pd.y}, vup[2] = {vu.x, vu.y}, vdn[2] = {vd.x, vd.y};
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                dxu[c] = fma(FD<R>::a(j), wu[R + c + j] - wu[R + c - j], dxu[c]);
                dxp[c] = fma(FD<R>::a(j), wp[R + c + j] - wp[R + c - j], dxp[c]);
                dyv[c] = fma(FD<R>::a(j), vup[c] - vdn[c], dyv[c]);
                dyp[c] = fma(FD<R>::a(j), pup[c] - pdn[c], dyp[c]);
            }
        }
        double pp[3][2] = {{0, 0}, {0, 0}, {0, 0}}, aa[3][2] = {{0, 0}, {0, 0}, {0, 0}};
        if constexpr (MODE != MODE_FE)
#pragma unroll
            for (int f = 0; f < 3; ++f) {
                const double2 t = *reinterpret_cast<const double2*>(st + L::O_PW + f * PWT + own);
                pp[f][0] = t.x; pp[f][1] = t.y;
            }
        if constexpr (MODE == MODE_FINACC)
#pragma unroll
            for (int f = 0; f < 3; ++f) {
                const double2 t = *reinterpret_cast<const double2*>(st + L::O_PW + (3 + f) * PWT + own);
                aa[f][0] = t.x; aa[f][1] = t.y;
            }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);          // this warp is done with stage s
        const double vv[2] = {vcen.x, vcen.y};
        double o[3][2];
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            const double fp = -fma(A.sx, dxu[c], A.sy * dyv[c]);
            const double fu = -A.sx * dxp[c];
            const double fv = -A.sy * dyp[c];
            o[0][c] = combine<MODE>(pp[0][c], wp[R + c], fp, aa[0][c], A.cf, A.wh);
            o[1][c] = combine<MODE>(pp[1][c], wu[R + c], fu, aa[1][c], A.cf, A.wh);
            o[2][c] = combine<MODE>(pp[2][c], vv[c], fv, aa[2][c], A.cf, A.wh);
            if constexpr (MODE == MODE_FIN0 || MODE == MODE_FINACC)
                bad |= !isfinite(o[0][c]) || !isfinite(o[1][c]) || !isfinite(o[2][c]);
        }
        const int64_t go = (int64_t)(ys + i * TY + ty) * nx + x0 + 2 * tx;   // slab-local row
#pragma unroll
        for (int f = 0; f < 3; ++f)
            *reinterpret_cast<double2*>(A.O[f] + go) = make_double2(o[f][0], o[f][1]);
    }
    if constexpr (MODE == MODE_FIN0 || MODE == MODE_FINACC)
        if (bad && A.nonfinite) *A.nonfinite = 1;
}

}  // namespace tma
}  // namespace gbs

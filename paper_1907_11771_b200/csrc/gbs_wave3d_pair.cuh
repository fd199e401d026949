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
// and S_v: each stencil value u_a(x') is recomputed as fma(cfA, S_v(x'), P_u(x')),
// exactly the operation the single-step kernel performs at x', and every sum is
// formed in the same order -- so the pair kernel is bit-identical to two
// launches of wave3d_step(_tma) (tested), while moving 32 B read + 32 B write
// per point for two substeps instead of 96 B (LF + LF).
//
// Outputs go to buffers distinct from P and S (their halos are read by
// neighbouring CTAs): LF writes y_{n+1} -> (Au, Av) and y_{n+2} -> (Bu, Bv);
// FIN writes only the accumulator (Bu, Bv).
//
// Pipeline (per CTA: 64x16 tile, 16 consumer warps x 2 points + 1 producer
// warp), stage for iteration i (plane z = z0 + i) carries:
//   tiles of S_u, S_v, P_u at plane z (centre column with y-halo + x strips, as
//   in gbs_wave3d_tma.cuh), the centre boxes of S_u, S_v, P_u at plane z + R
//   (fronts of the two register queues, lap(S_u) and lap(u_a) along z), P_v at
//   plane z, and the accumulator at plane z (FINACC).
#pragma once

#include "gbs_wave3d_tma.cuh"

namespace gbs {
namespace tma {

template <int R, int MODEB>
struct PairLayout {
    static constexpr int SH = TY + 2 * R;
    static constexpr int NACC = (MODEB == MODE_FINACC) ? 2 : 0;
    static constexpr int D = (MODEB == MODE_FINACC) ? 2 : 3;
    static constexpr int CENTER = SH * TX;
    static constexpr int STRIP = TY * R;
    static constexpr int TILE = CENTER + 2 * STRIP;
    static constexpr int PWT = TY * TX;
    // stage: 3 tiles | 3 fronts | P_v | acc (NACC)
    static constexpr int STAGE = 3 * TILE + (4 + NACC) * PWT;
    static constexpr size_t bytes = (size_t)D * STAGE * 8 + (2 * D) * 8;
    static constexpr uint32_t stage_bytes = STAGE * 8;
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
    const double* Su; const double* Sv; const double* Pu;   // for the register-queue warm-up
    int nx, ny, nz, zchunk;
    int64_t plane;
    double sx2, sy2, sz2;
    double cfA, cfB, wh;
    int* nonfinite;
};

template <int R, int MODEB, bool SLAB>
__global__ void __launch_bounds__(512, 1)
wave3d_pair_tma(const __grid_constant__ PairMaps M, const PairArgs A, const int zbase) {
    using L = PairLayout<R, MODEB>;
    constexpr int D = L::D, TILE = L::TILE, PWT = L::PWT, STAGE = L::STAGE;
    extern __shared__ __align__(128) double smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)D * STAGE);
    uint64_t* empty = full + D;

    const int tx = threadIdx.x, ty = threadIdx.y, lane = tx;
    const int nx = A.nx, ny = A.ny, nz = A.nz;
    const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
    const int z0 = blockIdx.z * A.zchunk;
    const int niter = min(A.zchunk, nz - z0);
    auto zc = [&](int z) -> int {
        if constexpr (SLAB) return z + zbase;
        else return wrap_once(z, nz);
    };

    if (ty == 0 && lane == 0) {
        for (int s = 0; s < D; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], TY); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    // Producer = lane 0 of warp 0 (a dedicated 17th warp would be allocated as 20
    // warps and cap the consumers at 96 registers).  Stage i is issued at the top
    // of iteration i - D + 1, after its slot's previous use (iteration i - D) has
    // been released by all 16 warps.
    const bool producer = (ty == 0 && lane == 0);
    auto issue_stage = [&](int i) {
        const CUtensorMap* maps[3][3] = {{&M.su_a, &M.su_b, &M.su_c}, {&M.sv_a, &M.sv_b, &M.sv_c},
                                         {&M.pu_a, &M.pu_b, &M.pu_c}};
        const int ytop = wrap_any(y0 - R, ny), ybot = wrap_any(y0 + TY, ny);
        const int xl = wrap_any(x0 - R, nx), xr = wrap_any(x0 + TX, nx);
        const int s = i % D;
        if (i >= D) mbar_wait(&empty[s], (uint32_t)(((i / D) - 1) & 1));
        mbar_expect_tx(&full[s], L::stage_bytes);
        double* st = smem + (size_t)s * STAGE;
        const int z = zc(z0 + i), zf = zc(z0 + i + R);
#pragma unroll
        for (int f = 0; f < 3; ++f) {
            double* t = st + f * TILE;
            tma_load_3d(t, maps[f][1], x0, ytop, z, &full[s]);
            tma_load_3d(t + R * TX, maps[f][0], x0, y0, z, &full[s]);
            tma_load_3d(t + (R + TY) * TX, maps[f][1], x0, ybot, z, &full[s]);
            tma_load_3d(t + L::CENTER, maps[f][2], xl, y0, z, &full[s]);
            tma_load_3d(t + L::CENTER + L::STRIP, maps[f][2], xr, y0, z, &full[s]);
            tma_load_3d(st + 3 * TILE + f * PWT, maps[f][0], x0, y0, zf, &full[s]);   // front
        }
        tma_load_3d(st + 3 * TILE + 3 * PWT, &M.pv, x0, y0, z, &full[s]);
        if constexpr (MODEB == MODE_FINACC) {
            tma_load_3d(st + 3 * TILE + 4 * PWT, &M.acc_u, x0, y0, z, &full[s]);
            tma_load_3d(st + 3 * TILE + 5 * PWT, &M.acc_v, x0, y0, z, &full[s]);
        }
    };
    if (producer) {
        prefetch_map(&M.su_a); prefetch_map(&M.su_b); prefetch_map(&M.su_c);
        prefetch_map(&M.sv_a); prefetch_map(&M.sv_b); prefetch_map(&M.sv_c);
        prefetch_map(&M.pu_a); prefetch_map(&M.pu_b); prefetch_map(&M.pu_c); prefetch_map(&M.pv);
        if constexpr (MODEB == MODE_FINACC) { prefetch_map(&M.acc_u); prefetch_map(&M.acc_v); }
        for (int i = 0; i < D - 1 && i < niter; ++i) issue_stage(i);
    }

    // ===================== all 16 warps compute =====================
    const int64_t plane = A.plane;
    const int64_t own = (int64_t)(y0 + ty) * nx + x0 + 2 * tx;
    auto zoff = [&](int z) -> int64_t {
        if constexpr (SLAB) return (int64_t)z * plane;
        else return (int64_t)wrap_once(z, nz) * plane;
    };
    using V = Vec<2>;
    V qs[2 * R + 1], qa[2 * R + 1];          // S_u and u_a at z-R .. z+R (own points)
#pragma unroll
    for (int j = 0; j < 2 * R; ++j) {
        const int64_t o = zoff(z0 - R + j) + own;
        qs[j] = V::ld(A.Su + o);
        const V sv = V::ld(A.Sv + o), pu = V::ld(A.Pu + o);
#pragma unroll
        for (int v = 0; v < 2; ++v) qa[j].v[v] = fma(A.cfA, sv.v[v], pu.v[v]);
    }

    bool bad = false;
    for (int i = 0; i < niter; ++i) {
        const int s = i % D;
        if (producer && i + D - 1 < niter) issue_stage(i + D - 1);
        mbar_wait(&full[s], (uint32_t)((i / D) & 1));
        double* st = smem + (size_t)s * STAGE;
        const double* tS = st;                  // S_u tile
        const double* tV = st + TILE;           // S_v tile
        double* tP = st + 2 * TILE;             // P_u tile, turned into the u_a tile below
        const double* fr = st + 3 * TILE + ty * TX + 2 * tx;   // fronts + pointwise, own column
        {
            const double2 fs = *reinterpret_cast<const double2*>(fr);
            const double2 fv = *reinterpret_cast<const double2*>(fr + PWT);
            const double2 fp = *reinterpret_cast<const double2*>(fr + 2 * PWT);
            qs[2 * R].v[0] = fs.x; qs[2 * R].v[1] = fs.y;
            qa[2 * R].v[0] = fma(A.cfA, fv.x, fp.x);
            qa[2 * R].v[1] = fma(A.cfA, fv.y, fp.y);
        }
        // u_a = fma(cfA, S_v, P_u) over the whole tile (halo included), once, in place
        {
            const double2* v2 = reinterpret_cast<const double2*>(tV);
            double2* p2 = reinterpret_cast<double2*>(tP);
            for (int e = ty * 32 + tx; e < TILE / 2; e += 32 * TY) {
                const double2 a = v2[e], b = p2[e];
                p2[e] = make_double2(fma(A.cfA, a.x, b.x), fma(A.cfA, a.y, b.y));
            }
        }
        __syncthreads();
        // x windows (columns 2tx - R .. 2tx + R + 1) of S_u and u_a
        double xs[2 * R + 2], xa[2 * R + 2];
#pragma unroll
        for (int k = 0; k <= R; ++k) {
            const int col = 2 * tx - R + 2 * k;
            const int off = col < 0 ? L::CENTER + ty * R + (col + R)
                          : col >= TX ? L::CENTER + L::STRIP + ty * R + (col - TX)
                                      : (R + ty) * TX + col;
            const double2 a = *reinterpret_cast<const double2*>(tS + off);
            const double2 c = *reinterpret_cast<const double2*>(tP + off);
            xs[2 * k] = a.x; xs[2 * k + 1] = a.y;
            xa[2 * k] = c.x; xa[2 * k + 1] = c.y;
        }
        const int crow = (R + ty) * TX + 2 * tx;
        double lsx[2], lsy[2], lsz[2], lax[2], lay[2], laz[2];
#pragma unroll
        for (int v = 0; v < 2; ++v) {
            const double cs = xs[R + v], ca = xa[R + v];
            lsx[v] = FD<R>::b0() * cs; lsy[v] = FD<R>::b0() * cs; lsz[v] = FD<R>::b0() * cs;
            lax[v] = FD<R>::b0() * ca; lay[v] = FD<R>::b0() * ca; laz[v] = FD<R>::b0() * ca;
        }
#pragma unroll
        for (int j = 1; j <= R; ++j) {
            const double2 su = *reinterpret_cast<const double2*>(tS + crow - j * TX);
            const double2 sd = *reinterpret_cast<const double2*>(tS + crow + j * TX);
            const double2 au = *reinterpret_cast<const double2*>(tP + crow - j * TX);
            const double2 ad = *reinterpret_cast<const double2*>(tP + crow + j * TX);
            const double su2[2] = {su.x, su.y}, sd2[2] = {sd.x, sd.y};
            const double au2[2] = {au.x, au.y}, ad2[2] = {ad.x, ad.y};
#pragma unroll
            for (int v = 0; v < 2; ++v) {
                lsx[v] = fma(FD<R>::b(j), xs[R + v + j] + xs[R + v - j], lsx[v]);
                lsy[v] = fma(FD<R>::b(j), sd2[v] + su2[v], lsy[v]);
                lsz[v] = fma(FD<R>::b(j), qs[R + j].v[v] + qs[R - j].v[v], lsz[v]);
                lax[v] = fma(FD<R>::b(j), xa[R + v + j] + xa[R + v - j], lax[v]);
                lay[v] = fma(FD<R>::b(j), ad2[v] + au2[v], lay[v]);
                laz[v] = fma(FD<R>::b(j), qa[R + j].v[v] + qa[R - j].v[v], laz[v]);
            }
        }
        const double* pvp = st + 3 * TILE + 3 * PWT + ty * TX + 2 * tx;
        const double2 pv = *reinterpret_cast<const double2*>(pvp);
        double2 accu = make_double2(0, 0), accv = make_double2(0, 0);
        if constexpr (MODEB == MODE_FINACC) {
            accu = *reinterpret_cast<const double2*>(pvp + PWT);
            accv = *reinterpret_cast<const double2*>(pvp + 2 * PWT);
        }
        // centre values of S_v for step B (from the S_v tile)
        const double2 svc = *reinterpret_cast<const double2*>(tV + crow);
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        const double pvv[2] = {pv.x, pv.y}, svv[2] = {svc.x, svc.y};
        const double acu[2] = {accu.x, accu.y}, acv[2] = {accv.x, accv.y};
        double ua[2], va[2], ub[2], vb[2];
#pragma unroll
        for (int v = 0; v < 2; ++v) {
            const double lapS = fma(A.sx2, lsx[v], fma(A.sy2, lsy[v], A.sz2 * lsz[v]));
            const double lapA = fma(A.sx2, lax[v], fma(A.sy2, lay[v], A.sz2 * laz[v]));
            ua[v] = xa[R + v];                                   // = fma(cfA, S_v, P_u): step A, u
            va[v] = combine<MODE_LF>(pvv[v], svv[v], lapS, 0.0, A.cfA, 0.0);      // step A, v
            ub[v] = combine<MODEB>(xs[R + v], ua[v], va[v], acu[v], A.cfB, A.wh);  // step B, u
            vb[v] = combine<MODEB>(svv[v], va[v], lapA, acv[v], A.cfB, A.wh);      // step B, v
            if constexpr (MODEB != MODE_LF) bad |= !isfinite(ub[v]) || !isfinite(vb[v]);
        }
        const int64_t o = zoff(z0 + i) + own;
        if constexpr (MODEB == MODE_LF) {
            *reinterpret_cast<double2*>(A.Au + o) = make_double2(ua[0], ua[1]);
            *reinterpret_cast<double2*>(A.Av + o) = make_double2(va[0], va[1]);
        }
        *reinterpret_cast<double2*>(A.Bu + o) = make_double2(ub[0], ub[1]);
        *reinterpret_cast<double2*>(A.Bv + o) = make_double2(vb[0], vb[1]);
#pragma unroll
        for (int j = 0; j < 2 * R; ++j) { qs[j] = qs[j + 1]; qa[j] = qa[j + 1]; }
    }
    if constexpr (MODEB != MODE_LF)
        if (bad && A.nonfinite) *A.nonfinite = 1;
}

}  // namespace tma
}  // namespace gbs

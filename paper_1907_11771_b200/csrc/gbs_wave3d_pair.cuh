// gbs_wave3d_pair.cuh -- two consecutive GBS substeps of the 3-D wave in one
// HBM pass (temporal blocking), TMA-fed.
//
// The u-component of a leap-frog step is pointwise (u_t = v):
//     u_{n+1} = u_{n-1} + 2h v_n            (Eq. (1) row 2)
// so the launch that produces v_n can also produce u_{n+1} in its epilogue, and
// the next launch receives the u-level one step ahead, U = u_{n+1}, already
// formed.  A launch of this kernel starts from
//     P_v = v_{n-1},  S = (S_u, S_v) = y_n,  U = u_{n+1}
// and computes
//   step A (LF):  v_{n+1} = P_v + cfA lap(S_u)                       -> Av (LF)
//   step B  LF :  u_{n+2} = S_u + cfB v_{n+1}                        -> Bu
//                 v_{n+2} = S_v + cfB lap(U)                         -> Bv
//                 u_{n+3} = U + cfA v_{n+2}   (the next launch's U)  -> Cu
//           FIN:  acc (+)= wh (S_u + U + cfB v_{n+1})                 (averaging and
//                 acc (+)= wh (S_v + v_{n+1} + cfB lap(U))             weighted sum,
//                                                                      PAPER.md:92, 109-115)
// Every value is formed by exactly the operation the single-substep kernel
// performs for it (fma(cf, f, p) for LF, wh (p + s + cf f) for FIN) with the
// sums of the Laplacian in the same order, so a sequence run through this
// kernel is bit-identical to one run substep by substep (tested).
// Per point: reads S_u, U, S_v, P_v (32 B), writes Av, Bu, Bv, Cu (32 B) for
// two substeps (96 B single-step); FIN reads 32 (+16 acc) and writes 16.
//
// In-place rules (host side): Av may alias P_v and Bv may alias S_v (both are
// read only at the thread's own points, a stage before they are written); Bu
// and Cu must not alias S_u or U (their halos are read by neighbouring CTAs).
//
// Pipeline: 64x16 tile, 8 warps, each thread owns a 2x2 block of points (two
// rows, two consecutive x).  Lane 0 of warp 0 issues the TMA boxes of plane
// z + D - 1 while plane z is computed: per stage the S_u and U tiles of plane z
// (centre column with y halos + two x strips, five boxes each; x/y stencils),
// the S_u and U centre boxes of plane z + R (fronts of the two register queues
// that carry the z stencils), and the own-point boxes S_v, P_v (and the
// accumulator) of plane z.  D = 3 stages (the two-stage version waited on the
// TMA barrier ~23% of the time, profiles/r01_ncu_pair_c5_src.txt).
// L2 policies (PairArgs::hint, default 11): the z+R centre boxes are loaded
// evict_last (re-read R planes later as the tile centre), the own-point boxes
// evict_first, and the outputs are streaming stores -- 10% fewer DRAM reads
// (profiles/r01_ncu_pair6_c5.txt).
#pragma once

#include "gbs_wave3d_tma.cuh"

namespace gbs {
namespace tma {

// MODE_FEA (this kernel only): the forward-Euler substep fused with the first step of one
// leap-frog chain, from the two stencil fields u_0 (the S_u slot) and v_0 (the U slot):
//   v_1 = v_0 + h lap(u_0), u_1 = u_0 + h v_0, u_2 = u_0 + 2h v_1        (FE, bit-exact)
//   lap(u_1) = lap(u_0) + h lap(v_0)                    (linearity: u_1 is never formed at
//   v_2 = v_0 + 2h lap(u_1), u_3 = u_1 + 2h v_2          its neighbours; rounding-level change)
// outputs Av = v_2, Bu = u_3 (chain A after its first step), Bv = v_1, Cu = u_2 (chain B's
// start): 16 B read + 32 B written per point instead of the FE's 40 + the first half's 32.
constexpr int MODE_FEA = 4;

template <int R, int MODEB>
struct PairLayout {
    static constexpr int SH = TY + 2 * R;
    static constexpr bool FEA = MODEB == MODE_FEA;
    static constexpr int NACC = (MODEB == MODE_FINACC) ? 2 : 0;
    static constexpr int NPW = FEA ? 0 : 2;                // S_v, P_v boxes
    static constexpr int D = FEA ? 5 : 3;                  // TMA stages
    static constexpr int CENTER = SH * TX;
    static constexpr int STRIP = TY * R;
    static constexpr int TILE = CENTER + 2 * STRIP;
    static constexpr int PWT = TY * TX;
    // stage: S_u tile (z) | U tile (z) | S_u centre (z+R) | U centre (z+R) |
    //        S_v centre (z) | P_v centre (z) | accumulator u, v (z, FINACC)
    static constexpr int O_UT = TILE, O_SUF = 2 * TILE, O_UF = 2 * TILE + PWT;
    static constexpr int O_SV = 2 * TILE + 2 * PWT, O_PV = 2 * TILE + 3 * PWT, O_AC = 2 * TILE + 4 * PWT;
    static constexpr int STAGE = 2 * TILE + (2 + NPW + NACC) * PWT;
    static constexpr size_t stage_doubles = (size_t)D * STAGE;
    static constexpr size_t bytes = stage_doubles * 8 + (2 * D + 1) * 8;
    static constexpr uint32_t stage_bytes = STAGE * 8;
    static_assert((TILE * 8) % 128 == 0 && (PWT * 8) % 128 == 0, "TMA destinations need 128 B alignment");
};

struct PairMaps {
    CUtensorMap su_a, su_b, su_c;     // S_u: TXxTY, TXxR, RxTY boxes
    CUtensorMap u_a, u_b, u_c;        // U
    CUtensorMap sv, pv, acc_u, acc_v; // TXxTY
};

struct PairArgs {
    double* Av;                       // v_{n+1} (LF)
    double* Bu; double* Bv;           // y_{n+2} (LF) or the accumulator (FIN)
    double* Cu;                       // u_{n+3} (LF)
    const double* Su; const double* U;
    int nx, ny, nz, zchunk;
    int zlo, zhi;                     // planes [zlo, zhi) of the slab this launch computes
    int zskip;                        // planes skipped after the first chunk (Wave3DArgs::zskip)
    int64_t plane;
    double sx2, sy2, sz2;
    double cfA, cfB, wh;
    int* nonfinite;
    int band;                         // launch order of the x-y tiles (tile_of)
    int hint;                         // L2 policy bits (experiment): 1 fronts evict_last,
                                      // 2 pointwise evict_first, 4 tiles evict_first, 8 .cs stores
};

template <int R, int MODEB, bool SLAB, bool PEER = false>
__global__ void __launch_bounds__(256, 1)
wave3d_pair_tma(const __grid_constant__ PairMaps M, const PairArgs A, const int zbase, const PeerPush P) {
    using L = PairLayout<R, MODEB>;
    constexpr int D = L::D, STAGE = L::STAGE;
    constexpr int NW = TY / 2;                 // 8 warps; each thread owns 2 x 2 points
    constexpr int Q = 2 * R + 1;
    extern __shared__ __align__(128) double smem[];
    double* stages = smem;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::stage_doubles);
    uint64_t* empty = full + D;

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

    const uint64_t pol_last = policy_evict_last(), pol_first = policy_evict_first();
    auto ld = [&](void* dst, const CUtensorMap* m, int x, int y, int z, uint64_t* bar, int bit, uint64_t pol) {
        if (A.hint & bit) tma_load_3d_hint(dst, m, x, y, z, bar, pol);
        else tma_load_3d(dst, m, x, y, z, bar);
    };
    auto load_tile = [&](double* dst, const CUtensorMap* a, const CUtensorMap* b, const CUtensorMap* c, int z,
                         uint64_t* bar) {
        ld(dst, b, x0, ytop, z, bar, 4, pol_first);
        ld(dst + R * TX, a, x0, y0, z, bar, 4, pol_first);
        ld(dst + (R + TY) * TX, b, x0, ybot, z, bar, 4, pol_first);
        ld(dst + L::CENTER, c, xl, y0, z, bar, 4, pol_first);
        ld(dst + L::CENTER + L::STRIP, c, xr, y0, z, bar, 4, pol_first);
    };
    auto issue_stage = [&](int i) {
        const int s = i % D;
        if (i >= D) mbar_wait(&empty[s], (uint32_t)(((i / D) - 1) & 1));
        mbar_expect_tx(&full[s], L::stage_bytes);
        double* st = stages + (size_t)s * STAGE;
        const int z = zc(z0 + i), zf = zc(z0 + i + R);
        load_tile(st, &M.su_a, &M.su_b, &M.su_c, z, &full[s]);
        load_tile(st + L::O_UT, &M.u_a, &M.u_b, &M.u_c, z, &full[s]);
        ld(st + L::O_SUF, &M.su_a, x0, y0, zf, &full[s], 1, pol_last);
        ld(st + L::O_UF, &M.u_a, x0, y0, zf, &full[s], 1, pol_last);
        if constexpr (!L::FEA) {
            ld(st + L::O_SV, &M.sv, x0, y0, z, &full[s], 2, pol_first);
            ld(st + L::O_PV, &M.pv, x0, y0, z, &full[s], 2, pol_first);
        }
        if constexpr (MODEB == MODE_FINACC) {
            ld(st + L::O_AC, &M.acc_u, x0, y0, z, &full[s], 2, pol_first);
            ld(st + L::O_AC + L::PWT, &M.acc_v, x0, y0, z, &full[s], 2, pol_first);
        }
    };

    const bool face = z0 < R || z0 + niter > nz - R;     // reads ghost planes / owns face planes
    if (producer) {
        for (int s = 0; s < D; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], NW); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        if constexpr (PEER) if (face) peer_wait(P);
    }
    __syncthreads();
    if (producer) {
        // the TMA (async proxy) reads of peer-pushed ghost planes are ordered after the
        // acquire by this thread's own proxy fence (the acquire ran on this thread too)
        if constexpr (PEER) asm volatile("fence.proxy.async.global;" ::: "memory");
        prefetch_map(&M.su_a); prefetch_map(&M.su_b); prefetch_map(&M.su_c);
        prefetch_map(&M.u_a); prefetch_map(&M.u_b); prefetch_map(&M.u_c);
        if constexpr (!L::FEA) { prefetch_map(&M.sv); prefetch_map(&M.pv); }
        if constexpr (MODEB == MODE_FINACC) { prefetch_map(&M.acc_u); prefetch_map(&M.acc_v); }
        for (int i = 0; i < D - 1 && i < niter; ++i) issue_stage(i);
    }
    // register queues of S_u and U at planes z-R .. z+R; point index 2*row + col
    double qs[Q][4], qa[Q][4];
#pragma unroll
    for (int j = 0; j < 2 * R; ++j) {
        const int64_t oz = zoff(z0 - R + j);
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            const int64_t o = oz + own + (int64_t)r * nx;
            // ghost planes may be peer-pushed memory: coherent loads (not .nc) under PEER
            const double2 su = PEER ? ld_relaxed_sys2(A.Su + o) : __ldg(reinterpret_cast<const double2*>(A.Su + o));
            const double2 uu = PEER ? ld_relaxed_sys2(A.U + o) : __ldg(reinterpret_cast<const double2*>(A.U + o));
            qs[j][2 * r] = su.x; qs[j][2 * r + 1] = su.y;
            qa[j][2 * r] = uu.x; qa[j][2 * r + 1] = uu.y;
        }
    }

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
                if (k == R / 2) {                   // the thread's own points: already in the queue
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
        double csv[4], cpv[4], cau[4] = {0, 0, 0, 0}, cav[4] = {0, 0, 0, 0};
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            const int po = (r0 + r) * TX + 2 * tx;                      // own column in a centre box
            const double2 fs = *reinterpret_cast<const double2*>(st + L::O_SUF + po);
            const double2 fu = *reinterpret_cast<const double2*>(st + L::O_UF + po);
            qs[2 * R][2 * r] = fs.x; qs[2 * R][2 * r + 1] = fs.y;
            qa[2 * R][2 * r] = fu.x; qa[2 * R][2 * r + 1] = fu.y;
            if constexpr (!L::FEA) {
                const double2 a = *reinterpret_cast<const double2*>(st + L::O_SV + po);
                const double2 b = *reinterpret_cast<const double2*>(st + L::O_PV + po);
                csv[2 * r] = a.x; csv[2 * r + 1] = a.y; cpv[2 * r] = b.x; cpv[2 * r + 1] = b.y;
            }
            if constexpr (MODEB == MODE_FINACC) {
                const double2 c = *reinterpret_cast<const double2*>(st + L::O_AC + po);
                const double2 d = *reinterpret_cast<const double2*>(st + L::O_AC + L::PWT + po);
                cau[2 * r] = c.x; cau[2 * r + 1] = c.y; cav[2 * r] = d.x; cav[2 * r + 1] = d.y;
            }
        }
        double lapS[4], lapU[4], xs_c[4], xu_c[4];
        lap4(st, qs, lapS, xs_c);                               // S_u tile, plane z
        lap4(st + L::O_UT, qa, lapU, xu_c);                     // U tile, plane z
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);                  // this warp is done with stage s
        double va[4], ub[4], vb[4], uc[4];
        if constexpr (L::FEA) {
            // S_u = u_0, U = v_0; cfA = h, cfB = 2h.  Outputs: va = v_2, ub = u_3, vb = v_1, uc = u_2
#pragma unroll
            for (int p = 0; p < 4; ++p) {
                const double u0 = xs_c[p], v0 = xu_c[p];
                vb[p] = combine<MODE_FE>(0.0, v0, lapS[p], 0.0, A.cfA, 0.0);        // v_1
                const double u1 = combine<MODE_FE>(0.0, u0, v0, 0.0, A.cfA, 0.0);   // u_1
                uc[p] = combine<MODE_LF>(u0, 0.0, vb[p], 0.0, A.cfB, 0.0);         // u_2
                const double lap1 = fma(A.cfA, lapU[p], lapS[p]);                   // lap(u_1)
                va[p] = combine<MODE_LF>(v0, 0.0, lap1, 0.0, A.cfB, 0.0);           // v_2
                ub[p] = combine<MODE_LF>(u1, 0.0, va[p], 0.0, A.cfB, 0.0);          // u_3
            }
        } else {
#pragma unroll
            for (int p = 0; p < 4; ++p) {
                va[p] = combine<MODE_LF>(cpv[p], csv[p], lapS[p], 0.0, A.cfA, 0.0);     // v_{n+1}
                ub[p] = combine<MODEB>(xs_c[p], xu_c[p], va[p], cau[p], A.cfB, A.wh);   // u_{n+2} / acc_u
                vb[p] = combine<MODEB>(csv[p], va[p], lapU[p], cav[p], A.cfB, A.wh);    // v_{n+2} / acc_v
                if constexpr (MODEB == MODE_LF) uc[p] = combine<MODE_LF>(xu_c[p], 0.0, vb[p], 0.0, A.cfA, 0.0);
                else bad |= !isfinite(ub[p]) || !isfinite(vb[p]);
            }
        }
        const int64_t oz = zoff(z0 + i);
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            const int64_t o = oz + own + (int64_t)r * nx;
            if (A.hint & 8) {
                if constexpr (MODEB == MODE_LF || L::FEA) {
                    __stcs(reinterpret_cast<double2*>(A.Av + o), make_double2(va[2 * r], va[2 * r + 1]));
                    __stcs(reinterpret_cast<double2*>(A.Cu + o), make_double2(uc[2 * r], uc[2 * r + 1]));
                }
                __stcs(reinterpret_cast<double2*>(A.Bu + o), make_double2(ub[2 * r], ub[2 * r + 1]));
                __stcs(reinterpret_cast<double2*>(A.Bv + o), make_double2(vb[2 * r], vb[2 * r + 1]));
                continue;
            }
            if constexpr (MODEB == MODE_LF || L::FEA) {
                *reinterpret_cast<double2*>(A.Av + o) = make_double2(va[2 * r], va[2 * r + 1]);
                *reinterpret_cast<double2*>(A.Cu + o) = make_double2(uc[2 * r], uc[2 * r + 1]);
            }
            *reinterpret_cast<double2*>(A.Bu + o) = make_double2(ub[2 * r], ub[2 * r + 1]);
            *reinterpret_cast<double2*>(A.Bv + o) = make_double2(vb[2 * r], vb[2 * r + 1]);
        }
        if constexpr (PEER) {
            // the u-levels read with stencils by the next launch: B_u (or the accumulator's u,
            // the next macro step's Y) and C_u
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                const int64_t xy = own + (int64_t)r * nx;
                peer_push2<R>(P, 0, z0 + i, plane, xy, ub[2 * r], ub[2 * r + 1]);
                if constexpr (MODEB == MODE_LF) peer_push2<R>(P, 1, z0 + i, plane, xy, uc[2 * r], uc[2 * r + 1]);
            }
        }
#pragma unroll
        for (int j = 0; j < 2 * R; ++j)
#pragma unroll
            for (int p = 0; p < 4; ++p) { qs[j][p] = qs[j + 1][p]; qa[j][p] = qa[j + 1][p]; }
    }
    if constexpr (PEER) {
        // one cumulative system fence per CTA after the barrier (the kernel boundary orders it
        // before the epoch signal)
        if (face) {
            __syncthreads();
            if (tx == 0 && ty == 0) __threadfence_system();
        }
    }
    if constexpr (MODEB != MODE_LF && !L::FEA)
        if (bad && A.nonfinite) *A.nonfinite = 1;
}

}  // namespace tma
}  // namespace gbs

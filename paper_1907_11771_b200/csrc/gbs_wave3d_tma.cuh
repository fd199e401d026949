// gbs_wave3d_tma.cuh -- 3-D wave substep kernel fed by the Tensor Memory
// Accelerator (cp.async.bulk.tensor, SASS UTMALDG) through a D-stage
// full/empty mbarrier pipeline with a dedicated producer warp.
//
// Same arithmetic, operand order and modes as gbs::wave3d_step
// (gbs_kernels.cuh), so the two kernels agree bit for bit: one launch is one
// FE / LF / final substep of one GBS sequence (Eq. (1), lines 85-98),
// the FIN modes fused with the averaging and the weighted accumulate
// (PAPER.md:109-115, 221-225).
//
// Why: the register-prefetch kernel keeps only about one plane of loads in
// flight per SM (1 CTA x 512 threads at 128 registers), which caps it near 78%
// of the copy bandwidth.  Here one producer thread issues 5 + NP tensor boxes
// per plane, up to D planes ahead of the 16 consumer warps, so the bytes in
// flight no longer depend on the register budget.
//
// Tile: TX = 64 (x) by TY = 16 (y) points, 16 consumer warps of 32 threads x 2
// points + 1 producer warp.  Per plane the u tile is five boxes that never
// overlap and never cross the periodic boundary (the grid is a multiple of the
// tile, so a wrapped halo box is simply a box at the wrapped coordinate):
//   centre column [TY + 2R][TX]: top halo (TX x R), centre (TX x TY), bottom halo (TX x R)
//   x strips [TY][R]: left (R x TY at x0 - R), right (R x TY at x0 + TX)
// Shared memory: ring[R + D] of those tiles (plane z is the x/y stencil at
// iteration z and the register-queue front at iteration z - R) and pw[D][NP]
// TX x TY tiles of the pointwise streams (v of the current level, u and v of
// the previous level, the accumulator for FINACC).
#pragma once

#include <cuda.h>

#include "gbs_kernels.cuh"

namespace gbs {
namespace tma {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int x, int y, int z, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
        : "memory");
}
// the same with an L2 eviction-priority policy (createpolicy)
__device__ __forceinline__ void tma_load_3d_hint(void* dst, const CUtensorMap* map, int x, int y, int z,
                                                 uint64_t* bar, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void prefetch_map(const CUtensorMap* map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

template <int MODE> struct NPW { static constexpr int v = (MODE == MODE_FE) ? 1 : (MODE == MODE_FINACC ? 5 : 3); };
template <int MODE> struct Depth { static constexpr int v = (MODE == MODE_FINACC) ? 3 : 4; };

constexpr int TX = 64, TY = 16;

// ---------------------------------------------------------------------------
// Peer halo pushes (option "peer", slabbed 3-D two-substep path):
// the launch that produces a u-level also stores the r face planes of its slab straight
// into the neighbours' ghost planes (peer memory over NVLink across GPUs; the neighbouring
// slab's buffer in loopback), so no halo exchange runs between substeps.  Ordering by
// per-slab epochs: after every launch a one-thread kernel release-stores the launch's
// epoch into both neighbours' flags; a CTA whose planes touch a slab face (it reads ghost
// planes or pushes face planes) first waits until both neighbours have finished the
// previous launch -- that covers RAW (their pushes of this launch's inputs are complete)
// and WAR (they are done reading the ghost planes of the buffers this launch overwrites:
// with the rotating u-slots only the previous launch read them).
struct PeerPush {
    double* lo[2];                         // lower neighbour's field base (plane 0) per pushed output
    double* hi[2];                         // upper neighbour's
    const unsigned long long* wait_lo;     // this slab's flags, written by the neighbours
    const unsigned long long* wait_hi;
    unsigned long long epoch;              // this launch
    int nz;                                // planes per slab (all slabs equal)
};

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
// coherent (not .nc) 128-bit load of memory other GPUs may write during the kernel
__device__ __forceinline__ double2 ld_relaxed_sys2(const double* p) {
    double2 v;
    asm volatile("ld.relaxed.sys.global.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void peer_wait(const PeerPush& P) {
    const unsigned long long need = P.epoch - 1;
    while (ld_acquire_sys(P.wait_lo) < need || ld_acquire_sys(P.wait_hi) < need) __nanosleep(200);
    asm volatile("fence.proxy.async.global;" ::: "memory");    // TMA reads see the pushed planes
}
// the face copy of a double2 the thread stores at slab plane z (offset `xy` in the plane)
template <int R>
__device__ __forceinline__ void peer_push2(const PeerPush& P, int o, int z, int64_t plane, int64_t xy, double a,
                                           double b) {
    if (z < R) *reinterpret_cast<double2*>(P.lo[o] + (int64_t)(P.nz + z) * plane + xy) = make_double2(a, b);
    if (z >= P.nz - R) *reinterpret_cast<double2*>(P.hi[o] + (int64_t)(z - P.nz) * plane + xy) = make_double2(a, b);
}
template <int Unused = 0>
__global__ void peer_signal(unsigned long long* to_lo, unsigned long long* to_hi, unsigned long long epoch) {
    __threadfence_system();
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(to_lo), "l"(epoch) : "memory");
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(to_hi), "l"(epoch) : "memory");
}

// Launch order of the ntx x nty tiles of a plane (grid x = ntx * nty): bands of `band`
// x-tiles, x fastest inside a band, then y, then the next band.  band = ntx is plain
// row order.  Resident CTAs start in launch order and march z at the same rate, so two
// tiles k launches apart run ~k/148 of a CTA lifetime apart in z: the band keeps the
// y-neighbours (whose halo rows a tile reads from L2) band launches apart instead of ntx.
__device__ __forceinline__ void tile_of(int L, int ntx, int nty, int band, int& xt, int& yt) {
    const int per = band * nty;
    const int b = L / per, r = L - b * per;
    yt = r / band;
    xt = b * band + (r - yt * band);
}

template <int R, int MODE>
struct Layout {
    static constexpr int SH = TY + 2 * R;
    static constexpr int D = Depth<MODE>::v;
    static constexpr int RING = R + D;
    static constexpr int NP = NPW<MODE>::v;
    static constexpr int CENTER = SH * TX;                 // doubles of the centre column
    static constexpr int STRIP = TY * R;                   // doubles of one x strip
    static constexpr int TILE = CENTER + 2 * STRIP;        // doubles per u tile (128 B multiple)
    static constexpr int PWT = TY * TX;
    static constexpr size_t ring_doubles = (size_t)RING * TILE;
    static constexpr size_t pw_doubles = (size_t)D * NP * PWT;
    static constexpr size_t bytes = (ring_doubles + pw_doubles) * 8 + (2 * D + 1) * 8;
    static constexpr uint32_t tile_bytes = TILE * 8;
    static constexpr uint32_t stage_bytes = tile_bytes + NP * PWT * 8;
    static_assert((CENTER * 8) % 128 == 0 && (STRIP * 8) % 128 == 0, "TMA destinations need 128 B alignment");
};

// Tensor maps of one launch.  Each map is a 3-D view [nz_alloc][ny][nx] of one
// field buffer (ghost planes included in slab mode; z coordinate = z + zbase).
struct Maps {
    CUtensorMap su_a, su_b, su_c;      // u of the current level: TXxTY, TXxR, RxTY boxes
    CUtensorMap sv, pu, pv, au, av;    // TXxTY boxes
};

template <int R, int MODE, bool SLAB, bool PEER = false>
__global__ void __launch_bounds__(544, 1)
wave3d_step_tma(const __grid_constant__ Maps M, const Wave3DArgs A, const int zbase, const PeerPush P) {
    using L = Layout<R, MODE>;
    constexpr int D = L::D, RING = L::RING, NP = L::NP, TILE = L::TILE, PWT = L::PWT;
    extern __shared__ __align__(128) double smem[];
    double* ring = smem;
    double* pw = smem + L::ring_doubles;
    uint64_t* full = reinterpret_cast<uint64_t*>(pw + L::pw_doubles);
    uint64_t* empty = full + D;
    uint64_t* init = empty + D;

    const int tx = threadIdx.x, ty = threadIdx.y, lane = tx;
    const int nx = A.nx, ny = A.ny, nz = A.nz;
    int xt, yt;
    tile_of(blockIdx.x, nx / TX, ny / TY, A.band, xt, yt);
    const int x0 = xt * TX, y0 = yt * TY;
    const int z0 = A.zlo + blockIdx.z * A.zchunk + (blockIdx.z ? A.zskip : 0);
    const int niter = min(A.zchunk, A.zhi - z0);

    auto zc = [&](int z) -> int {              // tensor z coordinate of logical plane z
        if constexpr (SLAB) return z + zbase;
        else return wrap_once(z, nz);
    };

    const bool face = z0 < R || z0 + niter > nz - R;     // reads ghost planes / owns face planes
    if (ty == 0 && lane == 0) {
        for (int s = 0; s < D; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], TY); }
        mbar_init(init, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        if constexpr (PEER) if (face) peer_wait(P);
    }
    __syncthreads();

    if (ty == TY) {
        // ===================== producer warp =====================
        if (lane != 0) return;
        // peer-pushed ghost planes: thread (0,0) acquired the neighbours' flags before the
        // barrier; the TMA issuing thread orders its async-proxy reads after it itself
        if constexpr (PEER) asm volatile("fence.proxy.async.global;" ::: "memory");
        prefetch_map(&M.su_a); prefetch_map(&M.su_b); prefetch_map(&M.su_c); prefetch_map(&M.sv);
        if constexpr (MODE != MODE_FE) { prefetch_map(&M.pu); prefetch_map(&M.pv); }
        if constexpr (MODE == MODE_FINACC) { prefetch_map(&M.au); prefetch_map(&M.av); }
        const int ytop = wrap_any(y0 - R, ny), ybot = wrap_any(y0 + TY, ny);
        const int xl = wrap_any(x0 - R, nx), xr = wrap_any(x0 + TX, nx);
        const uint64_t pol_last = policy_evict_last(), pol_first = policy_evict_first();
        auto ld = [&](void* dst, const CUtensorMap* m, int x, int y, int z, uint64_t* bar, int bit, uint64_t pol) {
            if (A.hint & bit) tma_load_3d_hint(dst, m, x, y, z, bar, pol);
            else tma_load_3d(dst, m, x, y, z, bar);
        };
        auto issue_tile = [&](int p, uint64_t* bar) {
            double* t = ring + (size_t)(p % RING) * TILE;
            const int z = zc(z0 + p);
            ld(t, &M.su_b, x0, ytop, z, bar, 1, pol_last);
            ld(t + R * TX, &M.su_a, x0, y0, z, bar, 1, pol_last);
            ld(t + (R + TY) * TX, &M.su_b, x0, ybot, z, bar, 1, pol_last);
            ld(t + L::CENTER, &M.su_c, xl, y0, z, bar, 1, pol_last);
            ld(t + L::CENTER + L::STRIP, &M.su_c, xr, y0, z, bar, 1, pol_last);
        };
        mbar_expect_tx(init, R * L::tile_bytes);
        for (int p = 0; p < R; ++p) issue_tile(p, init);
        for (int i = 0; i < niter; ++i) {
            const int s = i % D;
            if (i >= D) mbar_wait(&empty[s], (uint32_t)(((i / D) - 1) & 1));
            mbar_expect_tx(&full[s], L::stage_bytes);
            issue_tile(i + R, &full[s]);
            double* p = pw + (size_t)s * NP * PWT;
            const int z = zc(z0 + i);
            ld(p, &M.sv, x0, y0, z, &full[s], 2, pol_first);
            if constexpr (MODE != MODE_FE) {
                ld(p + PWT, &M.pu, x0, y0, z, &full[s], 2, pol_first);
                ld(p + 2 * PWT, &M.pv, x0, y0, z, &full[s], 2, pol_first);
            }
            if constexpr (MODE == MODE_FINACC) {
                ld(p + 3 * PWT, &M.au, x0, y0, z, &full[s], 2, pol_first);
                ld(p + 4 * PWT, &M.av, x0, y0, z, &full[s], 2, pol_first);
            }
        }
        return;
    }

    // ===================== consumer warps =====================
    const int64_t plane = A.plane;
    const int64_t own = (int64_t)(y0 + ty) * nx + x0 + 2 * tx;
    auto zoff = [&](int z) -> int64_t {
        if constexpr (SLAB) return (int64_t)z * plane;
        else return (int64_t)wrap_once(z, nz) * plane;
    };
    using V = Vec<2>;
    V q[2 * R + 1];
#pragma unroll
    for (int j = 0; j < R; ++j)                  // planes z0-R .. z0-1 (coherent under PEER)
        if constexpr (PEER) {
            const double2 t = ld_relaxed_sys2(A.Su + zoff(z0 - R + j) + own);
            q[j].v[0] = t.x; q[j].v[1] = t.y;
        } else {
            q[j] = V::ld(A.Su + zoff(z0 - R + j) + own);
        }
    mbar_wait(init, 0);
#pragma unroll
    for (int j = 0; j < R; ++j) {
        const double2 t = *reinterpret_cast<const double2*>(ring + (size_t)j * TILE + (R + ty) * TX + 2 * tx);
        q[R + j].v[0] = t.x; q[R + j].v[1] = t.y;
    }

    bool bad = false;
    for (int i = 0; i < niter; ++i) {
        const int s = i % D;
        mbar_wait(&full[s], (uint32_t)((i / D) & 1));
        const double* tile = ring + (size_t)(i % RING) * TILE;               // plane z
        const double* front = ring + (size_t)((i + R) % RING) * TILE;        // plane z + R
        {
            const double2 f = *reinterpret_cast<const double2*>(front + (R + ty) * TX + 2 * tx);
            q[2 * R].v[0] = f.x; q[2 * R].v[1] = f.y;
        }
        // x window: columns 2tx - R .. 2tx + R + 1 (pairs from the centre column or a strip)
        double xw[2 * R + 2];
#pragma unroll
        for (int k = 0; k <= R; ++k) {
            if (k == R / 2) {                   // the thread's own points: already in the queue
                xw[2 * k] = q[R].v[0]; xw[2 * k + 1] = q[R].v[1];
                continue;
            }
            const int col = 2 * tx - R + 2 * k;
            const double* src = col < 0 ? tile + L::CENTER + ty * R + (col + R)
                              : col >= TX ? tile + L::CENTER + L::STRIP + ty * R + (col - TX)
                                          : tile + (R + ty) * TX + col;
            const double2 t = *reinterpret_cast<const double2*>(src);
            xw[2 * k] = t.x; xw[2 * k + 1] = t.y;
        }
        const double* crow = tile + (R + ty) * TX + 2 * tx;
        double lx[2], ly[2], lz[2];
#pragma unroll
        for (int v = 0; v < 2; ++v) {
            const double c = xw[R + v];
            lx[v] = FD<R>::b0() * c; ly[v] = FD<R>::b0() * c; lz[v] = FD<R>::b0() * c;
        }
#pragma unroll
        for (int j = 1; j <= R; ++j) {
            const double2 up = *reinterpret_cast<const double2*>(crow - j * TX);
            const double2 dn = *reinterpret_cast<const double2*>(crow + j * TX);
            const double upv[2] = {up.x, up.y}, dnv[2] = {dn.x, dn.y};
#pragma unroll
            for (int v = 0; v < 2; ++v) {
                lx[v] = fma(FD<R>::b(j), xw[R + v + j] + xw[R + v - j], lx[v]);
                ly[v] = fma(FD<R>::b(j), dnv[v] + upv[v], ly[v]);
                lz[v] = fma(FD<R>::b(j), q[R + j].v[v] + q[R - j].v[v], lz[v]);
            }
        }
        const double* pws = pw + (size_t)s * NP * PWT + ty * TX + 2 * tx;
        const double2 sv = *reinterpret_cast<const double2*>(pws);
        double2 pu = make_double2(0, 0), pv = make_double2(0, 0), au = make_double2(0, 0), av = make_double2(0, 0);
        if constexpr (MODE != MODE_FE) {
            pu = *reinterpret_cast<const double2*>(pws + PWT);
            pv = *reinterpret_cast<const double2*>(pws + 2 * PWT);
        }
        if constexpr (MODE == MODE_FINACC) {
            au = *reinterpret_cast<const double2*>(pws + 3 * PWT);
            av = *reinterpret_cast<const double2*>(pws + 4 * PWT);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);          // this warp is done with stage s
        const double svv[2] = {sv.x, sv.y}, puv[2] = {pu.x, pu.y}, pvv[2] = {pv.x, pv.y};
        const double auv[2] = {au.x, au.y}, avv[2] = {av.x, av.y};
        double ou[2], ov[2];
#pragma unroll
        for (int v = 0; v < 2; ++v) {
            const double lap = fma(A.sx2, lx[v], fma(A.sy2, ly[v], A.sz2 * lz[v]));
            ou[v] = combine<MODE>(puv[v], xw[R + v], svv[v], auv[v], A.cf, A.wh);
            ov[v] = combine<MODE>(pvv[v], svv[v], lap, avv[v], A.cf, A.wh);
            if constexpr (MODE == MODE_FIN0 || MODE == MODE_FINACC)
                bad |= !isfinite(ou[v]) || !isfinite(ov[v]);
        }
        const int64_t o = zoff(z0 + i) + own;
        const bool cs = A.hint & 8;
        auto put = [&](double* p, double a, double b) {
            if (cs) __stcs(reinterpret_cast<double2*>(p), make_double2(a, b));
            else *reinterpret_cast<double2*>(p) = make_double2(a, b);
        };
        put(A.Ou + o, ou[0], ou[1]);
        put(A.Ov + o, ov[0], ov[1]);
        if constexpr (PEER) peer_push2<R>(P, 0, z0 + i, plane, own, ou[0], ou[1]);
        if constexpr (MODE == MODE_FE) {
            // u_2 = u_0 + 2h v_1 (the next leap-frog step's pointwise u, formed exactly as
            // the single-step LF kernel forms it) for the two-substep kernel
            if (A.Xu) {
                const double x0v = combine<MODE_LF>(xw[R], 0.0, ov[0], 0.0, A.cf2, 0.0);
                const double x1v = combine<MODE_LF>(xw[R + 1], 0.0, ov[1], 0.0, A.cf2, 0.0);
                put(A.Xu + o, x0v, x1v);
                if constexpr (PEER) peer_push2<R>(P, 1, z0 + i, plane, own, x0v, x1v);
            }
        }
#pragma unroll
        for (int j = 0; j < 2 * R; ++j) q[j] = q[j + 1];
    }
    if constexpr (PEER) {
        // the CTA's face pushes are ordered before the next launch's epoch signal by the
        // kernel boundary; one cumulative system fence per CTA after the consumers' barrier
        if (face) {
            asm volatile("bar.sync 1, %0;" ::"n"(32 * TY) : "memory");
            if (tx == 0 && ty == 0) __threadfence_system();
        }
    }
    if constexpr (MODE == MODE_FIN0 || MODE == MODE_FINACC)
        if (bad && A.nonfinite) *A.nonfinite = 1;
}

}  // namespace tma
}  // namespace gbs

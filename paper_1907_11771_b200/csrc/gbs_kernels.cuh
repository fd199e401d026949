// gbs_kernels.cuh -- sm_100a kernels of the extrapolated GBS hot path.
//
// One kernel launch = one RHS-evaluating substep of one GBS sequence
// (Eq. (1), lines 85-98), fused with what surrounds it so that each
// substep is a single HBM pass:
//
//   MODE_FE     out = S + cf f(S)                       cf = h      (Eq. (1) row 1)
//   MODE_LF     out = P + cf f(S)                       cf = 2h     (Eq. (1) row 2;
//                                                        out may alias P: in place)
//   MODE_FIN0   acc = wh (P + S + cf f(S))              cf = h, wh = w_k / 2
//   MODE_FINACC acc = acc + wh (P + S + cf f(S))
//
// The FIN modes are the last LF step, the averaging (Eq. (1) row 3) and the
// weighted extrapolation sum in one pass: with
// y_{N+1} = y_{N-1} + 2h f(y_N),
//   (y_{N-1} + 2 y_N + y_{N+1}) / 4 = (y_{N-1} + y_N + h f(y_N)) / 2,
// so y_{N+1} is never stored.
//
// f is the centered periodic FD right-hand side of the PDE (BASELINE.json
// configs), grid spacing 1/s_d:
//   D1 u_i = s * sum_j a_j (u_{i+j} - u_{i-j}),  D2 u_i = s^2 (b0 u_i + sum_j b_j (u_{i+j} + u_{i-j}))
// with the standard centered Taylor weights (typed here independently of the
// oracle; parity tests compare the two).
//
// Layout: SoA fp64 [F][nz][ny][nx], x fastest.  Every thread owns VX
// consecutive x points (VX = 2 -> 128-bit loads/stores) and marches along the
// slowest axis (z in 3-D, y in 2-D) keeping a register queue of 2r+1 planes of
// the fields whose stencil crosses that axis; the in-plane neighbours come from
// a double-buffered shared-memory tile with an r-wide halo (one __syncthreads
// per plane).  Loads for plane z+1 are issued before plane z is computed.
// Periodicity: every shared-memory cell is filled from the wrapped global
// coordinate of its position, so ragged edge tiles and wrap-around need no
// special cases; threads outside the grid compute on wrapped data and do not
// store.  SLAB = true replaces the wrap along the slowest axis by ghost planes
// (z in [-r, nz_local + r) is valid memory), filled by the halo exchange.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace gbs {

enum { MODE_FE = 0, MODE_LF = 1, MODE_FIN0 = 2, MODE_FINACC = 3 };

// ---- centered Taylor weights ----------------------------------------------
template <int R> struct FD;
template <> struct FD<2> {
    __device__ static constexpr double a(int j) { return j == 1 ? 2.0 / 3.0 : -1.0 / 12.0; }
    __device__ static constexpr double b0() { return -5.0 / 2.0; }
    __device__ static constexpr double b(int j) { return j == 1 ? 4.0 / 3.0 : -1.0 / 12.0; }
};
template <> struct FD<4> {
    __device__ static constexpr double a(int j) {
        return j == 1 ? 4.0 / 5.0 : j == 2 ? -1.0 / 5.0 : j == 3 ? 4.0 / 105.0 : -1.0 / 280.0;
    }
    __device__ static constexpr double b0() { return -205.0 / 72.0; }
    __device__ static constexpr double b(int j) {
        return j == 1 ? 8.0 / 5.0 : j == 2 ? -1.0 / 5.0 : j == 3 ? 8.0 / 315.0 : -1.0 / 560.0;
    }
};

__device__ __forceinline__ int wrap_once(int i, int n) { return i < 0 ? i + n : (i >= n ? i - n : i); }
__device__ __forceinline__ int wrap_any(int i, int n) { i %= n; return i < 0 ? i + n : i; }

template <int VX> struct Vec;
template <> struct Vec<1> {
    double v[1];
    __device__ __forceinline__ static Vec ld(const double* p) { Vec r; r.v[0] = __ldg(p); return r; }
    __device__ __forceinline__ static Vec ldrw(const double* p) { Vec r; r.v[0] = *p; return r; }
    __device__ __forceinline__ void st(double* p) const { *p = v[0]; }
};
template <> struct Vec<2> {
    double v[2];
    __device__ __forceinline__ static Vec ld(const double* p) {
        double2 t = __ldg(reinterpret_cast<const double2*>(p)); Vec r; r.v[0] = t.x; r.v[1] = t.y; return r;
    }
    __device__ __forceinline__ static Vec ldrw(const double* p) {
        double2 t = *reinterpret_cast<const double2*>(p); Vec r; r.v[0] = t.x; r.v[1] = t.y; return r;
    }
    __device__ __forceinline__ void st(double* p) const {
        *reinterpret_cast<double2*>(p) = make_double2(v[0], v[1]);
    }
};

// Combine one field's value according to MODE (p: previous level, s: current
// level, f: RHS, a: accumulator).
template <int MODE>
__device__ __forceinline__ double combine(double p, double s, double f, double a, double cf, double wh) {
    if constexpr (MODE == MODE_FE) return fma(cf, f, s);
    else if constexpr (MODE == MODE_LF) return fma(cf, f, p);
    else if constexpr (MODE == MODE_FIN0) return wh * (p + s + cf * f);
    else return fma(wh, p + s + cf * f, a);
}

struct NonfiniteFlag { int* flag; };

// ===========================================================================
// 3-D scalar wave  u_t = v,  v_t = lap(u)  (FD order 2R), z-march.
//   S: current level (Su, Sv); P: previous level (Pu, Pv; unused in FE);
//   O: output (y_{n+1} for FE/LF, the accumulator for FIN*).
// ===========================================================================
struct Wave3DArgs {
    const double* Su; const double* Sv;
    const double* Pu; const double* Pv;
    double* Ou; double* Ov;
    int nx, ny, nz;          // local extents (nz = local slab thickness)
    int zchunk;
    int zlo, zhi;            // planes [zlo, zhi) of the slab this launch computes
    int64_t plane;           // nx * ny
    double sx2, sy2, sz2;    // squared inverse spacings
    double cf, wh;
    int* nonfinite;          // optional flag (FIN modes)
    double* Xu;              // optional (FE, TMA kernel): u_2 = S_u + cf2 * v_1, the first
    double cf2;              // leap-frog step's u-component, for the two-substep kernel
    int zskip;               // planes skipped after the first z-chunk (the two face bands of a
                             // slab in one launch); 0 = contiguous chunks
    int band;                // TMA kernels: launch order of the x-y tiles (tma::tile_of)
    int hint;                // TMA kernel L2 policy bits: 1 u tiles evict_last, 2 pointwise
                             // boxes evict_first, 8 streaming (.cs) stores
};

template <int R, int MODE, int VX, int BY, bool SLAB>
__global__ void __launch_bounds__(32 * BY)
wave3d_step(const Wave3DArgs A) {
    constexpr int TX = 32 * VX, TY = BY, NT = 32 * BY;
    constexpr int SW = TX + 2 * R, SH = TY + 2 * R;
    constexpr int NYH = 2 * R * (TX / VX);     // y-halo vectors per plane
    constexpr int NXH = 2 * R * TY;            // x-halo scalars per plane
    constexpr int HPT_Y = (NYH + NT - 1) / NT;
    constexpr int HPT_X = (NXH + NT - 1) / NT;
    constexpr bool READ_P = (MODE != MODE_FE);
    constexpr bool READ_A = (MODE == MODE_FINACC);
    __shared__ __align__(16) double sm[2][SH][SW];

    const int tx = threadIdx.x, ty = threadIdx.y, t = ty * 32 + tx;
    const int nx = A.nx, ny = A.ny, nz = A.nz;
    const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
    const int z0 = A.zlo + blockIdx.z * A.zchunk + (blockIdx.z ? A.zskip : 0);
    const int z1 = min(z0 + A.zchunk, A.zhi);
    const int64_t plane = A.plane;

    const int gx = wrap_any(x0 + tx * VX, nx);
    const int gy = wrap_any(y0 + ty, ny);
    const bool valid = (x0 + tx * VX < nx) && (y0 + ty < ny);
    const int64_t own = (int64_t)gy * nx + gx;

    // halo sources (in-plane offsets) and shared-memory destinations, fixed over z
    int64_t yh_src[HPT_Y]; int yh_dst[HPT_Y]; bool yh_on[HPT_Y];
#pragma unroll
    for (int i = 0; i < HPT_Y; ++i) {
        int e = t + i * NT;
        yh_on[i] = e < NYH;
        int r = e / (TX / VX), c = e % (TX / VX);
        int row = r < R ? r : TY + r;                     // smem row
        int gyy = wrap_any(y0 - R + row, ny);
        int gxx = wrap_any(x0 + c * VX, nx);
        yh_src[i] = (int64_t)gyy * nx + gxx;
        yh_dst[i] = row * SW + R + c * VX;
    }
    int64_t xh_src[HPT_X]; int xh_dst[HPT_X]; bool xh_on[HPT_X];
#pragma unroll
    for (int i = 0; i < HPT_X; ++i) {
        int e = t + i * NT;
        xh_on[i] = e < NXH;
        int r = e / (2 * R), c = e % (2 * R);
        int col = c < R ? c : TX + c;                     // smem column
        int gyy = wrap_any(y0 + r, ny);
        int gxx = wrap_any(x0 - R + col, nx);
        xh_src[i] = (int64_t)gyy * nx + gxx;
        xh_dst[i] = (R + r) * SW + col;
    }

    auto zoff = [&](int z) -> int64_t {
        if constexpr (SLAB) return (int64_t)z * plane;
        else return (int64_t)wrap_once(z, nz) * plane;
    };

    using V = Vec<VX>;
    V q[2 * R + 1];                 // u at z-R .. z+R (own points)
#pragma unroll
    for (int j = 0; j < 2 * R; ++j) q[j] = V::ld(A.Su + zoff(z0 - R + j) + own);

    // prefetch registers for the next plane
    V nf, npu, npv, nsv, nau, nav;
    V nyh[HPT_Y]; double nxh[HPT_X];
    auto load_plane = [&](int z) {
        const int64_t oz = zoff(z);
        nf = V::ld(A.Su + zoff(z + R) + own);
        nsv = V::ld(A.Sv + oz + own);
        if constexpr (READ_P) { npu = V::ldrw(A.Pu + oz + own); npv = V::ldrw(A.Pv + oz + own); }
        if constexpr (READ_A) { nau = V::ldrw(A.Ou + oz + own); nav = V::ldrw(A.Ov + oz + own); }
#pragma unroll
        for (int i = 0; i < HPT_Y; ++i) if (yh_on[i]) nyh[i] = V::ld(A.Su + oz + yh_src[i]);
#pragma unroll
        for (int i = 0; i < HPT_X; ++i) if (xh_on[i]) nxh[i] = __ldg(A.Su + oz + xh_src[i]);
    };
    if (z0 < z1) load_plane(z0);

    bool bad = false;
    for (int z = z0; z < z1; ++z) {
        const int buf = z & 1;
        q[2 * R] = nf;
        V cpu = npu, cpv = npv, csv = nsv, cau = nau, cav = nav;
        // shared tile of u at plane z
        double* s = &sm[buf][0][0];
#pragma unroll
        for (int v = 0; v < VX; ++v) s[(R + ty) * SW + R + tx * VX + v] = q[R].v[v];
#pragma unroll
        for (int i = 0; i < HPT_Y; ++i)
            if (yh_on[i]) {
#pragma unroll
                for (int v = 0; v < VX; ++v) s[yh_dst[i] + v] = nyh[i].v[v];
            }
#pragma unroll
        for (int i = 0; i < HPT_X; ++i) if (xh_on[i]) s[xh_dst[i]] = nxh[i];
        if (z + 1 < z1) load_plane(z + 1);
        __syncthreads();

        const int64_t oz = zoff(z);
        V ou, ov;
#pragma unroll
        for (int v = 0; v < VX; ++v) {
            const double c = q[R].v[v];
            const double* row = s + (R + ty) * SW + R + tx * VX + v;
            double lx = FD<R>::b0() * c, ly = FD<R>::b0() * c, lz = FD<R>::b0() * c;
#pragma unroll
            for (int j = 1; j <= R; ++j) {
                lx = fma(FD<R>::b(j), row[j] + row[-j], lx);
                ly = fma(FD<R>::b(j), row[j * SW] + row[-j * SW], ly);
                lz = fma(FD<R>::b(j), q[R + j].v[v] + q[R - j].v[v], lz);
            }
            const double lap = fma(A.sx2, lx, fma(A.sy2, ly, A.sz2 * lz));
            // u_t = v, v_t = lap(u)
            ou.v[v] = combine<MODE>(cpu.v[v], c, csv.v[v], cau.v[v], A.cf, A.wh);
            ov.v[v] = combine<MODE>(cpv.v[v], csv.v[v], lap, cav.v[v], A.cf, A.wh);
            if constexpr (MODE == MODE_FIN0 || MODE == MODE_FINACC)
                bad |= !isfinite(ou.v[v]) || !isfinite(ov.v[v]);
        }
        if (valid) {
            ou.st(A.Ou + oz + own);
            ov.st(A.Ov + oz + own);
        }
#pragma unroll
        for (int j = 0; j < 2 * R; ++j) q[j] = q[j + 1];
    }
    if constexpr (MODE == MODE_FIN0 || MODE == MODE_FINACC)
        if (bad && valid && A.nonfinite) *A.nonfinite = 1;
}

// ===========================================================================
// 2-D acoustics  p_t = -(u_x + v_y), u_t = -p_x, v_t = -p_y  (FD order 2R),
// y-march.  Register queues of p and v along y; p and u rows with x-halo in
// shared memory.  Fields of S/P/O: index 0 = p, 1 = u, 2 = v.
// ===========================================================================
struct Acoustic2DArgs {
    const double* S[3];
    const double* P[3];
    double* O[3];
    int nx, ny;              // local extents (ny = local slab thickness)
    int ychunk;
    int ylo, yhi;            // rows [ylo, yhi) of the slab this launch computes
    int yskip;               // rows skipped after the first y-chunk (both face bands in one launch)
    double sx, sy;           // inverse spacings
    double cf, wh;
    int* nonfinite;
};

template <int R, int MODE, int VX, int NT, bool SLAB>
__global__ void __launch_bounds__(NT)
acoustic2d_step(const Acoustic2DArgs A) {
    constexpr int TX = NT * VX;
    constexpr int SW = TX + 2 * R;
    constexpr bool READ_P = (MODE != MODE_FE);
    constexpr bool READ_A = (MODE == MODE_FINACC);
    __shared__ __align__(16) double sp[2][SW];
    __shared__ __align__(16) double su[2][SW];

    const int tx = threadIdx.x;
    const int nx = A.nx, ny = A.ny;
    const int x0 = blockIdx.x * TX;
    const int ys = A.ylo + blockIdx.y * A.ychunk + (blockIdx.y ? A.yskip : 0);
    const int ye = min(ys + A.ychunk, A.yhi);
    const int gx = wrap_any(x0 + tx * VX, nx);
    const bool valid = x0 + tx * VX < nx;
    // x-halo: threads 0..4R-1 load p (0..2R-1) and u (2R..4R-1) halo columns
    const bool hon = tx < 4 * R;
    const int hc = tx % (2 * R);
    const int hcol = hc < R ? hc : TX + hc;
    const int hgx = wrap_any(x0 - R + hcol, nx);
    const int hfield = tx < 2 * R ? 0 : 1;

    auto yoff = [&](int y) -> int64_t {
        if constexpr (SLAB) return (int64_t)y * nx;
        else return (int64_t)wrap_once(y, ny) * nx;
    };

    using V = Vec<VX>;
    V qp[2 * R + 1], qv[2 * R + 1];
#pragma unroll
    for (int j = 0; j < 2 * R; ++j) {
        const int64_t o = yoff(ys - R + j) + gx;
        qp[j] = V::ld(A.S[0] + o);
        qv[j] = V::ld(A.S[2] + o);
    }
    V nfp, nfv, nu, np0, np1, np2, na0, na1, na2;
    double nh = 0.0;
    auto load_row = [&](int y) {
        const int64_t oy = yoff(y);
        const int64_t of = yoff(y + R) + gx;
        nfp = V::ld(A.S[0] + of);
        nfv = V::ld(A.S[2] + of);
        nu = V::ld(A.S[1] + oy + gx);
        if constexpr (READ_P) {
            np0 = V::ldrw(A.P[0] + oy + gx); np1 = V::ldrw(A.P[1] + oy + gx); np2 = V::ldrw(A.P[2] + oy + gx);
        }
        if constexpr (READ_A) {
            na0 = V::ldrw(A.O[0] + oy + gx); na1 = V::ldrw(A.O[1] + oy + gx); na2 = V::ldrw(A.O[2] + oy + gx);
        }
        if (hon) nh = __ldg(A.S[hfield] + oy + hgx);
    };
    if (ys < ye) load_row(ys);

    bool bad = false;
    for (int y = ys; y < ye; ++y) {
        const int buf = y & 1;
        qp[2 * R] = nfp; qv[2 * R] = nfv;
        V cu = nu, c0 = np0, c1 = np1, c2 = np2, a0 = na0, a1 = na1, a2 = na2;
#pragma unroll
        for (int v = 0; v < VX; ++v) {
            sp[buf][R + tx * VX + v] = qp[R].v[v];
            su[buf][R + tx * VX + v] = cu.v[v];
        }
        if (hon) (hfield == 0 ? sp : su)[buf][hcol] = nh;
        if (y + 1 < ye) load_row(y + 1);
        __syncthreads();

        const int64_t oy = yoff(y) + gx;
        V o0, o1, o2;
#pragma unroll
        for (int v = 0; v < VX; ++v) {
            const double* rp = &sp[buf][R + tx * VX + v];
            const double* ru = &su[buf][R + tx * VX + v];
            double dxu = 0.0, dxp = 0.0, dyv = 0.0, dyp = 0.0;
#pragma unroll
            for (int j = 1; j <= R; ++j) {
                dxu = fma(FD<R>::a(j), ru[j] - ru[-j], dxu);
                dxp = fma(FD<R>::a(j), rp[j] - rp[-j], dxp);
                dyv = fma(FD<R>::a(j), qv[R + j].v[v] - qv[R - j].v[v], dyv);
                dyp = fma(FD<R>::a(j), qp[R + j].v[v] - qp[R - j].v[v], dyp);
            }
            const double fp = -fma(A.sx, dxu, A.sy * dyv);
            const double fu = -A.sx * dxp;
            const double fv = -A.sy * dyp;
            o0.v[v] = combine<MODE>(c0.v[v], qp[R].v[v], fp, a0.v[v], A.cf, A.wh);
            o1.v[v] = combine<MODE>(c1.v[v], cu.v[v], fu, a1.v[v], A.cf, A.wh);
            o2.v[v] = combine<MODE>(c2.v[v], qv[R].v[v], fv, a2.v[v], A.cf, A.wh);
            if constexpr (MODE == MODE_FIN0 || MODE == MODE_FINACC)
                bad |= !isfinite(o0.v[v]) || !isfinite(o1.v[v]) || !isfinite(o2.v[v]);
        }
        if (valid) {
            o0.st(A.O[0] + oy);
            o1.st(A.O[1] + oy);
            o2.st(A.O[2] + oy);
        }
#pragma unroll
        for (int j = 0; j < 2 * R; ++j) { qp[j] = qp[j + 1]; qv[j] = qv[j + 1]; }
    }
    if constexpr (MODE == MODE_FIN0 || MODE == MODE_FINACC)
        if (bad && valid && A.nonfinite) *A.nonfinite = 1;
}

// ===========================================================================
// Ghost rows/planes of a single slab from its own periodic opposite side (the
// 2-D two-substep kernels read 2r rows beyond their bands): for each listed
// field, ghosts [-g, 0) <- [n - g, n) and [n, n + g) <- [0, g), plane = points per row/plane.
// ===========================================================================
struct GhostFillArgs {
    double* f[6];            // field bases (interior row 0)
    int nf;
    int64_t n, g, plane;
};

static __global__ void __launch_bounds__(256) ghost_fill(const GhostFillArgs A) {
    const int64_t per = A.g * A.plane;                       // values per side per field
    const int which = blockIdx.y;                            // field
    double* base = A.f[which];
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < per; i += (int64_t)gridDim.x * blockDim.x) {
        base[i - per] = base[(A.n - A.g) * A.plane + i];     // below row 0 <- top rows
        base[A.n * A.plane + i] = base[i];                   // above row n-1 <- bottom rows
    }
}

// ===========================================================================
// 1-D advection  u_t = -u_x  (FD order 2R): one thread per point, shared tile
// with a wrapped r-halo.
// ===========================================================================
struct Adv1DArgs {
    const double* S; const double* P; double* O;
    int nx; double sx; double cf, wh; int* nonfinite;
};

// Spectral derivative (order 0) on grids beyond the cluster kernel, between cuFFT's D2Z and
// Z2D: spec[k] <- i s k spec[k] for 0 <= k < N/2 (s = 2 pi / (L N), the 1/N of the unnormalised
// inverse included), the Nyquist coefficient dropped (it has no odd derivative)
template <int Unused = 0>
__global__ void __launch_bounds__(256) spectral_ik(double2* spec, int n, double s) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k > n / 2) return;
    const double2 t = spec[k];
    const double m = s * (double)k;
    spec[k] = (k == n / 2) ? make_double2(0.0, 0.0) : make_double2(-m * t.y, m * t.x);
}

// the pointwise update of one substep from the spectral derivative du = u_x: f = -u_x
template <int MODE>
__global__ void __launch_bounds__(256) adv1d_spectral_update(const Adv1DArgs A, const double* du) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    if (x >= A.nx) return;
    const double f = -du[x];
    double p = 0.0, a = 0.0;
    if constexpr (MODE != MODE_FE) p = A.P[x];
    if constexpr (MODE == MODE_FINACC) a = A.O[x];
    const double o = combine<MODE>(p, A.S[x], f, a, A.cf, A.wh);
    A.O[x] = o;
    if constexpr (MODE == MODE_FIN0 || MODE == MODE_FINACC)
        if (!isfinite(o) && A.nonfinite) *A.nonfinite = 1;
}

template <int R, int MODE, int NT>
__global__ void __launch_bounds__(NT)
adv1d_step(const Adv1DArgs A) {
    __shared__ double s[NT + 2 * R];
    const int tx = threadIdx.x, nx = A.nx;
    const int x0 = blockIdx.x * NT;
    const int x = x0 + tx;
    const bool valid = x < nx;
    const int gx = wrap_any(x, nx);
    s[R + tx] = __ldg(A.S + gx);
    if (tx < 2 * R) {
        const int col = tx < R ? tx : NT + tx;
        s[col] = __ldg(A.S + wrap_any(x0 - R + col, nx));
    }
    __syncthreads();
    double d = 0.0;
#pragma unroll
    for (int j = 1; j <= R; ++j) d = fma(FD<R>::a(j), s[R + tx + j] - s[R + tx - j], d);
    const double f = -A.sx * d;
    if (!valid) return;
    double p = 0.0, a = 0.0;
    if constexpr (MODE != MODE_FE) p = A.P[x];
    if constexpr (MODE == MODE_FINACC) a = A.O[x];
    const double o = combine<MODE>(p, s[R + tx], f, a, A.cf, A.wh);
    A.O[x] = o;
    if constexpr (MODE == MODE_FIN0 || MODE == MODE_FINACC)
        if (!isfinite(o) && A.nonfinite) *A.nonfinite = 1;
}

}  // namespace gbs

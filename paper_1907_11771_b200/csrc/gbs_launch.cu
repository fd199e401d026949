// gbs_launch.cu -- device memory (state buffers, ghost planes, tensor maps) and
// every kernel launch: the per-substep kernels (register z/y-march, TMA-pipelined
// 3-D and 2-D, the two-substep 3-D kernel) over a plane range of a slab, and the
// whole-run thread-block-cluster kernel for small 1-D grids (FD and spectral).
#include <mutex>
#include <set>
#include <utility>

#include "gbs_internal.h"
#include "gbs_kernels.cuh"
#include "gbs_wave3d_tma.cuh"
#include "gbs_wave3d_pair.cuh"
#include "gbs_wave3d_half.cuh"
#include "gbs_acoustic2d_tma.cuh"
#include "gbs_acoustic2d_pair.cuh"
#include "gbs_adv1d_cluster.cuh"

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
typedef CUresult (*EncodeTiled_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiled_t encode_tiled() {
    static EncodeTiled_t fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (EncodeTiled_t)p;
    }
    return fn;
}

// 3-D fp64 view [dz][ny][nx] at base with box (bx, by, 1)
static bool make_map(CUtensorMap* m, double* base, int64_t nx, int64_t ny, int64_t dz, int bx, int by) {
    EncodeTiled_t enc = encode_tiled();
    if (!enc) return false;
    cuuint64_t dims[3] = {(cuuint64_t)nx, (cuuint64_t)ny, (cuuint64_t)dz};
    cuuint64_t strides[2] = {(cuuint64_t)nx * 8, (cuuint64_t)(nx * ny) * 8};
    cuuint32_t box[3] = {(cuuint32_t)bx, (cuuint32_t)by, 1};
    cuuint32_t es[3] = {1, 1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Layout of the state: slabs of the slowest axis with ghost planes, the number of
// buffers per slab; no device memory yet (ensure_buffers allocates on first use, from
// a caller-bound workspace when there is one).
static int launch_spectral_step(gbs_ctx* c, const gbs::Adv1DArgs& a, int mode);   // below

int alloc_state(gbs_ctx* c) {
    int rc0 = spectral_setup(c);     // plans before any graph capture (they allocate)
    if (rc0) return rc0;
    int nloc = c->loopback;
    int64_t total_slabs = (int64_t)c->slabs * nloc;
    int64_t nzl = c->nslow / total_slabs;
    // 2-D TMA grids keep 2r ghost rows even on one slab (a self-exchange refreshes them): the
    // two-substep 2-D kernels read 2r rows beyond their bands and never wrap in y
    const bool ac2d_tma = c->pde == GBS_ACOUSTIC2D && c->n[0] % gbs::tma::TX == 0 && nzl % gbs::tma::TY == 0 &&
                          nzl >= 4 * c->R;
    c->ghost = ac2d_tma ? 2 * c->R : (total_slabs > 1 ? c->R : 0);
    c->field_stride = (nzl + 2 * c->ghost) * c->plane;
    // the TMA (and two-substep) kernels need the grid to be a multiple of their tile so
    // halo boxes never cross the wrap; the two-substep kernels need 4 level buffers
    // (2-D acoustics: x a multiple of the tile width, each slab's rows a multiple of its height)
    c->tma_grid = (c->pde == GBS_WAVE3D && c->n[0] % gbs::tma::TX == 0 && c->n[1] % gbs::tma::TY == 0) ||
                  (c->pde == GBS_ACOUSTIC2D && c->n[0] % gbs::tma::TX == 0 && nzl % gbs::tma::TY == 0);
    c->nbuf = c->tma_grid ? 6 : 4;
    c->slab.assign(nloc, Slab());
    for (int v = 0; v < nloc; ++v) {
        Slab& s = c->slab[v];
        int64_t gidx = (int64_t)c->my_slab * nloc + v;
        s.z0 = gidx * nzl;
        s.nz = nzl;
    }
    c->buffers_ready = false;
    if (!c->d_flag) {
        CU(c, cudaMalloc(&c->d_flag, sizeof(int)));
        CU(c, cudaMemsetAsync(c->d_flag, 0, sizeof(int), c->stream));
    }
    return GBS_OK;
}

static int64_t buffer_bytes(const gbs_ctx* c) {
    const int64_t b = (int64_t)sizeof(double) * c->F * c->field_stride;
    return (b + 255) / 256 * 256;                        // 256-byte aligned carve-out
}

int64_t state_bytes(const gbs_ctx* c) { return (int64_t)c->slab.size() * c->nbuf * buffer_bytes(c); }

int ensure_buffers(gbs_ctx* c) {
    if (c->buffers_ready) return GBS_OK;
    const int64_t bb = buffer_bytes(c);
    if (c->ws_ptr && c->ws_bytes < state_bytes(c))
        return fail(c, GBS_E_INVAL, "bound workspace of %lld bytes < %lld needed by this layout",
                    (long long)c->ws_bytes, (long long)state_bytes(c));
    char* ws = static_cast<char*>(c->ws_ptr);
    for (size_t v = 0; v < c->slab.size(); ++v) {
        Slab& s = c->slab[v];
        const int64_t nzl = s.nz;
        for (int b = 0; b < c->nbuf; ++b) {
            if (ws) {
                s.buf[b] = reinterpret_cast<double*>(ws + (int64_t)(v * c->nbuf + b) * bb);
            } else if (cudaMalloc(&s.buf[b], (size_t)bb) != cudaSuccess) {
                s.buf[b] = nullptr;
                free_state(c);                                // all buffers or none
                return fail(c, GBS_E_NOMEM, "cudaMalloc of %lld bytes failed", (long long)bb);
            }
            CU(c, cudaMemsetAsync(s.buf[b], 0, (size_t)bb, c->stream));
        }
        // TMA kernels: the grid must be a multiple of the tile so halo boxes never cross the wrap
        s.tma_ok = false;
        if (c->tma_grid) {
            bool ok = true;
            const int64_t dz = nzl + 2 * c->ghost;
            // 3-D: views [dz][ny][nx]; 2-D: [1][ny_alloc][nx] (the slow axis is y)
            const int64_t vy = c->pde == GBS_WAVE3D ? c->n[1] : dz, vz = c->pde == GBS_WAVE3D ? dz : 1;
            for (int b = 0; b < c->nbuf && ok; ++b)
                for (int f = 0; f < c->F && ok; ++f) {
                    double* base = s.buf[b] + (int64_t)f * c->field_stride;
                    ok = make_map(&s.tm[b][f][0], base, c->n[0], vy, vz, gbs::tma::TX, gbs::tma::TY) &&
                         make_map(&s.tm[b][f][1], base, c->n[0], vy, vz, gbs::tma::TX, c->R) &&
                         make_map(&s.tm[b][f][2], base, c->n[0], vy, vz, c->R, gbs::tma::TY);
                    if (ok && c->pde == GBS_WAVE3D && c->n[1] % gbs::tma::TYH_TALL == 0)   // half kernel, tall tiles
                        ok = make_map(&s.tm[b][f][3], base, c->n[0], vy, vz, gbs::tma::TX, gbs::tma::TYH_TALL) &&
                             make_map(&s.tm[b][f][4], base, c->n[0], vy, vz, c->R, gbs::tma::TYH_TALL);
                    if (ok && c->pde == GBS_ACOUSTIC2D) {   // the chain kernels' boxes (Ac2PairMaps)
                        const int BH = gbs::tma::AC2_BH;
                        ok = make_map(&s.tm[b][f][3], base, c->n[0], vy, vz, gbs::tma::TX, BH) &&
                             make_map(&s.tm[b][f][4], base, c->n[0], vy, vz, c->R, BH) &&
                             make_map(&s.tm[b][f][5], base, c->n[0], vy, vz, gbs::tma::TX, BH + 2 * c->R) &&
                             make_map(&s.tm[b][f][6], base, c->n[0], vy, vz, c->R, BH + 2 * c->R) &&
                             make_map(&s.tm[b][f][7], base, c->n[0], vy, vz, gbs::tma::TX, BH + 4 * c->R) &&
                             make_map(&s.tm[b][f][8], base, c->n[0], vy, vz, c->R, BH + 4 * c->R);
                    }
                }
            s.tma_ok = ok;
        }
    }
    c->buffers_ready = true;
    return GBS_OK;
}

void free_state(gbs_ctx* c) {
    for (auto& s : c->slab)
        for (int b = 0; b < 6; ++b) {
            if (s.buf[b] && !c->ws_ptr) cudaFree(s.buf[b]);
            s.buf[b] = nullptr;
        }
    c->buffers_ready = false;
}

// Opt a kernel into its dynamic shared memory once per (device, kernel): the attribute
// belongs to the device's context, so a process driving several devices sets it on each.
static cudaError_t ensure_smem(const void* fn, size_t bytes) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    static std::mutex mu;
    static std::set<std::pair<int, const void*>> done;
    std::lock_guard<std::mutex> lock(mu);
    if (done.count({dev, fn})) return cudaSuccess;
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e == cudaSuccess) done.insert({dev, fn});
    return e;
}

template <int R, int MODE, bool SLAB>
static void launch_wave3d(const gbs::Wave3DArgs& a, dim3 grid, bool vx2, cudaStream_t st) {
    if (vx2) gbs::wave3d_step<R, MODE, 2, 16, SLAB><<<grid, dim3(32, 16), 0, st>>>(a);
    else gbs::wave3d_step<R, MODE, 1, 16, SLAB><<<grid, dim3(32, 16), 0, st>>>(a);
}
// peer: the face pushes of this launch (slab layouts; the FE kernel and the pair kernel only)
template <int R, int MODE, bool SLAB>
static cudaError_t launch_wave3d_tma(const gbs::tma::Maps& m, const gbs::Wave3DArgs& a, int zbase, dim3 grid,
                                     cudaStream_t st, const gbs::tma::PeerPush* peer) {
    using L = gbs::tma::Layout<R, MODE>;
    const dim3 block(32, gbs::tma::TY + 1);
    if constexpr (SLAB && MODE == gbs::MODE_FE) {
        if (peer) {
            auto k = gbs::tma::wave3d_step_tma<R, MODE, true, true>;
            cudaError_t e = ensure_smem(reinterpret_cast<const void*>(k), L::bytes);
            if (e != cudaSuccess) return e;
            k<<<grid, block, L::bytes, st>>>(m, a, zbase, *peer);
            return cudaSuccess;
        }
    }
    if (peer) return cudaErrorNotSupported;
    cudaError_t e = ensure_smem(reinterpret_cast<const void*>(gbs::tma::wave3d_step_tma<R, MODE, SLAB>), L::bytes);
    if (e != cudaSuccess) return e;
    gbs::tma::wave3d_step_tma<R, MODE, SLAB><<<grid, block, L::bytes, st>>>(m, a, zbase, gbs::tma::PeerPush{});
    return cudaSuccess;
}
template <int R, int MODEB, bool SLAB>
static cudaError_t launch_pair_tma(const gbs::tma::PairMaps& m, const gbs::tma::PairArgs& a, int zbase, dim3 grid,
                                   cudaStream_t st, const gbs::tma::PeerPush* peer) {
    using L = gbs::tma::PairLayout<R, MODEB>;
    const dim3 block(32, gbs::tma::TY / 2);
    if constexpr (SLAB) {
        if (peer) {
            auto k = gbs::tma::wave3d_pair_tma<R, MODEB, true, true>;
            cudaError_t e = ensure_smem(reinterpret_cast<const void*>(k), L::bytes);
            if (e != cudaSuccess) return e;
            k<<<grid, block, L::bytes, st>>>(m, a, zbase, *peer);
            return cudaSuccess;
        }
    }
    if (peer) return cudaErrorNotSupported;
    cudaError_t e = ensure_smem(reinterpret_cast<const void*>(gbs::tma::wave3d_pair_tma<R, MODEB, SLAB>), L::bytes);
    if (e != cudaSuccess) return e;
    gbs::tma::wave3d_pair_tma<R, MODEB, SLAB><<<grid, block, L::bytes, st>>>(m, a, zbase, gbs::tma::PeerPush{});
    return cudaSuccess;
}

// ---------------------------------------------------------------------------
// peer halo pushes: neighbour addresses and flags
// ---------------------------------------------------------------------------
int peer_eligible(const gbs_ctx* c, bool multi_gpu) {
    if (c->pde != GBS_WAVE3D) return 0;
    if (!(c->use_fuse && c->use_bulk && c->tma_grid)) return 0;     // the FE + two-substep path
    if (multi_gpu) return c->world > 1 && c->slabs > 1 && c->groups == 1 && c->loopback == 1;
    return c->world == 1 && c->loopback > 1;
}

double* peer_field(gbs_ctx* c, int v, int side, int b, int f) {
    if (c->loopback > 1) {
        const int n = c->loopback;
        return field_ptr(c, c->slab[(v + (side ? 1 : -1) + n) % n], b, f);
    }
    const char* mine = reinterpret_cast<const char*>(field_ptr(c, c->slab[0], b, f));
    return reinterpret_cast<double*>(c->peer_base[side] + (mine - static_cast<const char*>(c->ws_ptr)));
}

unsigned long long* peer_flag(gbs_ctx* c, int v, int which) {
    if (c->loopback > 1) return c->d_peer_flags + 2 * v + which;
    return reinterpret_cast<unsigned long long*>(static_cast<char*>(c->ws_ptr) + state_bytes(c)) + which;
}

// the flag of neighbour `side` that this slab's signal updates: the lower neighbour waits on
// its "from upper" flag, the upper one on its "from lower" flag
unsigned long long* peer_flag_remote(gbs_ctx* c, int v, int side) {
    if (c->loopback > 1) {
        const int n = c->loopback, w = (v + (side ? 1 : -1) + n) % n;
        return c->d_peer_flags + 2 * w + (side ? 0 : 1);
    }
    return reinterpret_cast<unsigned long long*>(c->peer_base[side] + state_bytes(c)) + (side ? 0 : 1);
}

// this launch's PeerPush for slab s (outputs o0, o1 with o.b < 0 = none), or nullptr
static const gbs::tma::PeerPush* make_peer(gbs_ctx* c, Slab& s, Slot o0, Slot o1, gbs::tma::PeerPush& P) {
    if (!c->peer_on) return nullptr;
    const int v = (int)(&s - c->slab.data());
    P = gbs::tma::PeerPush{};
    const Slot o[2] = {o0, o1};
    for (int k = 0; k < 2; ++k)
        if (o[k].b >= 0) {
            P.lo[k] = peer_field(c, v, 0, o[k].b, o[k].f);
            P.hi[k] = peer_field(c, v, 1, o[k].b, o[k].f);
        }
    P.wait_lo = peer_flag(c, v, 0);
    P.wait_hi = peer_flag(c, v, 1);
    P.epoch = c->peer_epoch;
    P.nz = (int)s.nz;
    return &P;
}
template <int R, int MODE, bool SLAB>
static cudaError_t launch_ac2d_tma(const gbs::tma::AcMaps& m, const gbs::Acoustic2DArgs& a, int ybase, dim3 grid,
                                   cudaStream_t st) {
    using L = gbs::tma::AcLayout<R, MODE>;
    cudaError_t e = ensure_smem(reinterpret_cast<const void*>(gbs::tma::acoustic2d_step_tma<R, MODE, SLAB>), L::bytes);
    if (e != cudaSuccess) return e;
    gbs::tma::acoustic2d_step_tma<R, MODE, SLAB><<<grid, dim3(32, gbs::tma::TY + 1), L::bytes, st>>>(m, a, ybase);
    return cudaSuccess;
}
// rows per CTA of the 2-D TMA kernel: a multiple of the tile height minimising
// (waves of one-CTA-per-SM) x (rows + ~2 tiles of pipeline fill)
static int ac2d_ychunk(int64_t xtiles, int64_t ny, int opt, int sms, int T = gbs::tma::TY) {
    if (opt > 0) return (int)std::min<int64_t>(ny, ((opt + T - 1) / T) * T);
    int64_t best = -1, bestc = T;
    for (int64_t yc = T; yc <= ny; yc += T) {
        const int64_t ctas = xtiles * ((ny + yc - 1) / yc);
        const int64_t cost = ((ctas + sms - 1) / sms) * (yc + 2 * T);
        if (best < 0 || cost < best) { best = cost; bestc = yc; }
    }
    return (int)bestc;
}
template <int R, int MODE, bool SLAB>
static void launch_ac2d(const gbs::Acoustic2DArgs& a, dim3 grid, bool vx2, cudaStream_t st) {
    if (vx2) gbs::acoustic2d_step<R, MODE, 2, 128, SLAB><<<grid, 128, 0, st>>>(a);
    else gbs::acoustic2d_step<R, MODE, 1, 128, SLAB><<<grid, 128, 0, st>>>(a);
}

// x-tiles per launch-order band of the 3-D TMA kernels (tma::tile_of): option "band"
// when it divides the tile count, else whole rows
static int tile_band(const gbs_ctx* c, int64_t ntx) {
    const int b = c->band_opt;
    return (b > 0 && ntx % b == 0) ? b : (int)ntx;
}

// gap > 0: the launch covers the two face bands [lo, lo + B) and [hi - B, hi) of a slab,
// B = (hi - lo - gap) / 2, as two chunks of B planes (rows) with `gap` skipped between them
static void face_chunks(int64_t lo, int64_t hi, int64_t gap, int& chunk, int& skip, unsigned& nchunks) {
    if (gap <= 0) { skip = 0; return; }
    chunk = (int)((hi - lo - gap) / 2);
    skip = (int)gap;
    nchunks = 2;
}

static int chunk_for(int64_t tiles, int64_t extent, int zchunk_opt) {
    if (zchunk_opt > 0) return (int)std::min<int64_t>(zchunk_opt, extent);
    // aim at >= ~16 resident waves of CTAs so the tail stays small, with
    // chunks of at least 32 planes so the 2r warm-up planes stay cheap
    const int64_t target = 148 * 2 * 16;
    int64_t chunks = std::max<int64_t>(1, (target + tiles - 1) / tiles);
    chunks = std::min<int64_t>(chunks, std::max<int64_t>(1, extent / 32));
    return (int)((extent + chunks - 1) / chunks);
}

// one substep over the planes [lo, hi) of slab s (lo = 0, hi = s.nz: the whole slab)
int launch_step(gbs_ctx* c, Slab& s, const StepOperands& op, int64_t lo, int64_t hi, int64_t gap) {
    // slab kernels read ghost planes refreshed from neighbours; one slab (2-D TMA grids keep
    // ghost rows for the two-substep kernels) wraps periodically like a plain grid
    const bool slab = c->ghost > 0 && c->slabs * c->loopback > 1;
    int* flag = op.flag ? c->d_flag : nullptr;
    if (c->pde == GBS_WAVE3D) {
        gbs::Wave3DArgs a{};
        a.Su = field_ptr(c, s, op.S, 0); a.Sv = field_ptr(c, s, op.S, 1);
        a.Pu = field_ptr(c, s, op.P, 0); a.Pv = field_ptr(c, s, op.P, 1);
        a.Ou = field_ptr(c, s, op.O, 0); a.Ov = field_ptr(c, s, op.O, 1);
        a.nx = (int)c->n[0]; a.ny = (int)c->n[1]; a.nz = (int)s.nz;
        a.plane = c->plane;
        const double sx = c->n[0] / c->len[0], sy = c->n[1] / c->len[1], sz = c->n[2] / c->len[2];
        a.sx2 = sx * sx; a.sy2 = sy * sy; a.sz2 = sz * sz;
        a.cf = op.cf; a.wh = op.wh; a.nonfinite = flag;
        a.Xu = op.xu.b >= 0 ? field_ptr(c, s, op.xu.b, op.xu.f) : nullptr;
        a.cf2 = op.cf2;
        const bool vx2 = (c->n[0] % 2) == 0;
        if (c->use_bulk && s.tma_ok) {
            int64_t tx = c->n[0] / gbs::tma::TX, ty = c->n[1] / gbs::tma::TY;
            a.zlo = (int)lo; a.zhi = (int)hi;
            a.zchunk = c->zchunk_opt > 0 ? (int)std::min<int64_t>(c->zchunk_opt, hi - lo)
                                         : (int)std::min<int64_t>(128, hi - lo);
            a.band = tile_band(c, tx);
            a.hint = c->hint_step_opt;
            dim3 grid((unsigned)(tx * ty), 1u, (unsigned)((hi - lo + a.zchunk - 1) / a.zchunk));
            face_chunks(lo, hi, gap, a.zchunk, a.zskip, grid.z);
            gbs::tma::Maps m;
            m.su_a = s.tm[op.S][0][0]; m.su_b = s.tm[op.S][0][1]; m.su_c = s.tm[op.S][0][2];
            m.sv = s.tm[op.S][1][0];
            m.pu = s.tm[op.P][0][0]; m.pv = s.tm[op.P][1][0];
            m.au = s.tm[op.O][0][0]; m.av = s.tm[op.O][1][0];
            const int zbase = (int)c->ghost;
            cudaError_t e = cudaSuccess;
            gbs::tma::PeerPush pp;
            const gbs::tma::PeerPush* peer = make_peer(c, s, Slot{op.O, 0}, op.xu, pp);
#define W3B(RR, SL)                                                                                   \
            switch (op.mode) {                                                                        \
                case gbs::MODE_FE: e = launch_wave3d_tma<RR, gbs::MODE_FE, SL>(m, a, zbase, grid, c->stream, peer); break;     \
                case gbs::MODE_LF: e = launch_wave3d_tma<RR, gbs::MODE_LF, SL>(m, a, zbase, grid, c->stream, peer); break;     \
                case gbs::MODE_FIN0: e = launch_wave3d_tma<RR, gbs::MODE_FIN0, SL>(m, a, zbase, grid, c->stream, peer); break; \
                default: e = launch_wave3d_tma<RR, gbs::MODE_FINACC, SL>(m, a, zbase, grid, c->stream, peer); break;           \
            }
            if (c->R == 2) { if (slab) { W3B(2, true) } else { W3B(2, false) } }
            else { if (slab) { W3B(4, true) } else { W3B(4, false) } }
#undef W3B
            if (e != cudaSuccess) return fail(c, GBS_E_CUDA, "bulk kernel setup: %s", cudaGetErrorString(e));
            c->launches++;
            e = cudaGetLastError();
            if (e != cudaSuccess) return fail(c, GBS_E_CUDA, "kernel launch failed: %s", cudaGetErrorString(e));
            return GBS_OK;
        }
        const int TX = vx2 ? 64 : 32, TY = 16;
        int64_t tx = (c->n[0] + TX - 1) / TX, ty = (c->n[1] + TY - 1) / TY;
        a.zlo = (int)lo; a.zhi = (int)hi;
        a.zchunk = chunk_for(tx * ty, hi - lo, c->zchunk_opt);
        dim3 grid((unsigned)tx, (unsigned)ty, (unsigned)((hi - lo + a.zchunk - 1) / a.zchunk));
        face_chunks(lo, hi, gap, a.zchunk, a.zskip, grid.z);
#define W3(RR, SL)                                                                   \
        switch (op.mode) {                                                           \
            case gbs::MODE_FE: launch_wave3d<RR, gbs::MODE_FE, SL>(a, grid, vx2, c->stream); break;   \
            case gbs::MODE_LF: launch_wave3d<RR, gbs::MODE_LF, SL>(a, grid, vx2, c->stream); break;   \
            case gbs::MODE_FIN0: launch_wave3d<RR, gbs::MODE_FIN0, SL>(a, grid, vx2, c->stream); break; \
            default: launch_wave3d<RR, gbs::MODE_FINACC, SL>(a, grid, vx2, c->stream); break;         \
        }
        if (c->R == 2) { if (slab) { W3(2, true) } else { W3(2, false) } }
        else { if (slab) { W3(4, true) } else { W3(4, false) } }
#undef W3
    } else if (c->pde == GBS_ACOUSTIC2D) {
        gbs::Acoustic2DArgs a{};
        for (int f = 0; f < 3; ++f) {
            a.S[f] = field_ptr(c, s, op.S, f);
            a.P[f] = field_ptr(c, s, op.P, f);
            a.O[f] = field_ptr(c, s, op.O, f);
        }
        a.nx = (int)c->n[0]; a.ny = (int)s.nz;
        a.sx = c->n[0] / c->len[0]; a.sy = c->n[1] / c->len[1];
        a.cf = op.cf; a.wh = op.wh; a.nonfinite = flag;
        if (c->use_bulk && s.tma_ok) {
            const int64_t xt = c->n[0] / gbs::tma::TX;
            a.ylo = (int)lo; a.yhi = (int)hi;
            a.ychunk = ac2d_ychunk(xt, hi - lo, c->zchunk_opt, c->sms);
            dim3 grid((unsigned)xt, (unsigned)((hi - lo + a.ychunk - 1) / a.ychunk));
            face_chunks(lo, hi, gap, a.ychunk, a.yskip, grid.y);
            gbs::tma::AcMaps m;
            for (int f = 0; f < 3; ++f) {
                m.s_a[f] = s.tm[op.S][f][0]; m.s_b[f] = s.tm[op.S][f][1]; m.s_c[f] = s.tm[op.S][f][2];
                m.p[f] = s.tm[op.P][f][0];
                m.acc[f] = s.tm[op.O][f][0];
            }
            const int ybase = (int)c->ghost;
            cudaError_t e = cudaSuccess;
#define A2B(RR, SL)                                                                                     \
            switch (op.mode) {                                                                          \
                case gbs::MODE_FE: e = launch_ac2d_tma<RR, gbs::MODE_FE, SL>(m, a, ybase, grid, c->stream); break;     \
                case gbs::MODE_LF: e = launch_ac2d_tma<RR, gbs::MODE_LF, SL>(m, a, ybase, grid, c->stream); break;     \
                case gbs::MODE_FIN0: e = launch_ac2d_tma<RR, gbs::MODE_FIN0, SL>(m, a, ybase, grid, c->stream); break; \
                default: e = launch_ac2d_tma<RR, gbs::MODE_FINACC, SL>(m, a, ybase, grid, c->stream); break;           \
            }
            if (c->R == 2) { if (slab) { A2B(2, true) } else { A2B(2, false) } }
            else { if (slab) { A2B(4, true) } else { A2B(4, false) } }
#undef A2B
            if (e != cudaSuccess) return fail(c, GBS_E_CUDA, "bulk kernel setup: %s", cudaGetErrorString(e));
            c->launches++;
            e = cudaGetLastError();
            if (e != cudaSuccess) return fail(c, GBS_E_CUDA, "kernel launch failed: %s", cudaGetErrorString(e));
            return GBS_OK;
        }
        const bool vx2 = (c->n[0] % 2) == 0;
        const int TX = vx2 ? 256 : 128;
        int64_t tx = (c->n[0] + TX - 1) / TX;
        a.ylo = (int)lo; a.yhi = (int)hi;
        a.ychunk = chunk_for(tx, hi - lo, c->zchunk_opt);
        dim3 grid((unsigned)tx, (unsigned)((hi - lo + a.ychunk - 1) / a.ychunk));
        face_chunks(lo, hi, gap, a.ychunk, a.yskip, grid.y);
#define A2(RR, SL)                                                                   \
        switch (op.mode) {                                                           \
            case gbs::MODE_FE: launch_ac2d<RR, gbs::MODE_FE, SL>(a, grid, vx2, c->stream); break;   \
            case gbs::MODE_LF: launch_ac2d<RR, gbs::MODE_LF, SL>(a, grid, vx2, c->stream); break;   \
            case gbs::MODE_FIN0: launch_ac2d<RR, gbs::MODE_FIN0, SL>(a, grid, vx2, c->stream); break; \
            default: launch_ac2d<RR, gbs::MODE_FINACC, SL>(a, grid, vx2, c->stream); break;         \
        }
        if (c->R == 2) { if (slab) { A2(2, true) } else { A2(2, false) } }
        else { if (slab) { A2(4, true) } else { A2(4, false) } }
#undef A2
    } else {
        gbs::Adv1DArgs a;
        a.S = field_ptr(c, s, op.S, 0); a.P = field_ptr(c, s, op.P, 0); a.O = field_ptr(c, s, op.O, 0);
        a.nx = (int)c->n[0]; a.sx = c->n[0] / c->len[0];
        a.cf = op.cf; a.wh = op.wh; a.nonfinite = flag;
        if (c->order == 0) {
            const int rc = launch_spectral_step(c, a, op.mode);
            if (rc) return rc;
            cudaError_t e = cudaGetLastError();
            if (e != cudaSuccess) return fail(c, GBS_E_CUDA, "kernel launch failed: %s", cudaGetErrorString(e));
            return GBS_OK;
        }
        constexpr int NT = 256;
        dim3 grid((unsigned)((c->n[0] + NT - 1) / NT));
#define A1(RR)                                                                            \
        switch (op.mode) {                                                                \
            case gbs::MODE_FE: gbs::adv1d_step<RR, gbs::MODE_FE, NT><<<grid, NT, 0, c->stream>>>(a); break;   \
            case gbs::MODE_LF: gbs::adv1d_step<RR, gbs::MODE_LF, NT><<<grid, NT, 0, c->stream>>>(a); break;   \
            case gbs::MODE_FIN0: gbs::adv1d_step<RR, gbs::MODE_FIN0, NT><<<grid, NT, 0, c->stream>>>(a); break; \
            default: gbs::adv1d_step<RR, gbs::MODE_FINACC, NT><<<grid, NT, 0, c->stream>>>(a); break;         \
        }
        if (c->R == 2) { A1(2) } else { A1(4) }
#undef A1
    }
    c->launches++;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(c, GBS_E_CUDA, "kernel launch failed: %s", cudaGetErrorString(e));
    return GBS_OK;
}

// the two-laplacian passes with both stencil fields fed through tile rings (wave3d_ring2):
// the fused FE + first chain step, and the LF + final pass
template <int R, int MODE, bool SLAB>
static cudaError_t launch_ring2_k(const gbs::tma::Ring2Maps& m, const gbs::tma::Ring2Args& a, int zbase, dim3 grid,
                                  cudaStream_t st) {
    using RL = gbs::tma::Ring2Layout<R, MODE>;
    auto k = gbs::tma::wave3d_ring2<R, MODE, SLAB>;
    cudaError_t e = ensure_smem(reinterpret_cast<const void*>(k), RL::bytes);
    if (e != cudaSuccess) return e;
    k<<<grid, dim3(32, gbs::tma::TY / 2), RL::bytes, st>>>(m, a, zbase);
    return cudaSuccess;
}

static int launch_ring2(gbs_ctx* c, Slab& s, const PairOperands& op, int64_t lo, int64_t hi, int64_t gap) {
    const bool slab = c->ghost > 0 && c->slabs * c->loopback > 1;
    const bool fea = op.modeB == gbs::tma::MODE_FEA;
    gbs::tma::Ring2Args a{};
    a.Su = field_ptr(c, s, op.Su.b, op.Su.f);
    a.U = field_ptr(c, s, op.U.b, op.U.f);
    if (fea) {
        a.A2 = field_ptr(c, s, op.Av.b, op.Av.f);
        a.A3 = field_ptr(c, s, op.Bu.b, op.Bu.f);
        a.A1 = field_ptr(c, s, op.Bv.b, op.Bv.f);
        a.A4 = field_ptr(c, s, op.Cu.b, op.Cu.f);
    } else {
        a.A3 = op.out_u ? op.out_u : field_ptr(c, s, op.Bu.b, 0);
        a.A1 = op.out_v ? op.out_v : field_ptr(c, s, op.Bu.b, 1);
    }
    a.nx = (int)c->n[0]; a.ny = (int)c->n[1]; a.nz = (int)s.nz;
    a.plane = c->plane;
    const double sx = c->n[0] / c->len[0], sy = c->n[1] / c->len[1], sz = c->n[2] / c->len[2];
    a.sx2 = sx * sx; a.sy2 = sy * sy; a.sz2 = sz * sz;
    a.cfA = op.cfA; a.cfB = op.cfB; a.wh = op.wh;
    a.nonfinite = op.flag ? c->d_flag : nullptr;
    a.zlo = (int)lo; a.zhi = (int)hi;
    const int64_t tiles = (c->n[0] / gbs::tma::TX) * (c->n[1] / gbs::tma::TY);
    const int zauto = tiles * ((hi - lo + 255) / 256) >= 8LL * c->sms ? 256 : 128;
    int zc = c->zchunk_pair_opt > 0 ? c->zchunk_pair_opt : c->zchunk_opt > 0 ? c->zchunk_opt : zauto;
    if (!fea && c->zchunk_fin_opt > 0) zc = c->zchunk_fin_opt;
    a.zchunk = (int)std::min<int64_t>(zc, hi - lo);
    a.band = tile_band(c, c->n[0] / gbs::tma::TX);
    a.hint = fea ? c->hint_opt : c->hint_fin_opt;
    dim3 grid((unsigned)tiles, 1u, (unsigned)((hi - lo + a.zchunk - 1) / a.zchunk));
    face_chunks(lo, hi, gap, a.zchunk, a.zskip, grid.z);
    gbs::tma::Ring2Maps m;
    m.u.x_a = s.tm[op.Su.b][op.Su.f][0]; m.u.x_b = s.tm[op.Su.b][op.Su.f][1]; m.u.x_c = s.tm[op.Su.b][op.Su.f][2];
    m.v.x_a = s.tm[op.U.b][op.U.f][0]; m.v.x_b = s.tm[op.U.b][op.U.f][1]; m.v.x_c = s.tm[op.U.b][op.U.f][2];
    if (!fea) {
        m.sv = s.tm[op.Sv.b][op.Sv.f][0];
        m.pv = s.tm[op.Pv.b][op.Pv.f][0];
        m.acc_u = s.tm[op.Bu.b][0][0];
        m.acc_v = s.tm[op.Bu.b][1][0];
    }
    const int zbase = (int)c->ghost;
    cudaError_t e = cudaSuccess;
#define RG(RR, SL)                                                                                  \
    switch (op.modeB) {                                                                             \
        case gbs::tma::MODE_FEA: e = launch_ring2_k<RR, gbs::tma::MODE_FEA, SL>(m, a, zbase, grid, c->stream); break; \
        case gbs::MODE_FIN0: e = launch_ring2_k<RR, gbs::MODE_FIN0, SL>(m, a, zbase, grid, c->stream); break;         \
        default: e = launch_ring2_k<RR, gbs::MODE_FINACC, SL>(m, a, zbase, grid, c->stream); break;                    \
    }
    if (c->R == 2) { if (slab) { RG(2, true) } else { RG(2, false) } }
    else { if (slab) { RG(4, true) } else { RG(4, false) } }
#undef RG
    if (e != cudaSuccess) return fail(c, GBS_E_CUDA, "ring2 kernel setup: %s", cudaGetErrorString(e));
    c->launches++;
    e = cudaGetLastError();
    if (e != cudaSuccess) return fail(c, GBS_E_CUDA, "kernel launch failed: %s", cudaGetErrorString(e));
    return GBS_OK;
}

int launch_pair(gbs_ctx* c, Slab& s, const PairOperands& op, int64_t lo, int64_t hi, int64_t gap) {
    if (!c->peer_on && ((op.modeB == gbs::tma::MODE_FEA && c->fea_ring) ||
                        ((op.modeB == gbs::MODE_FIN0 || op.modeB == gbs::MODE_FINACC) && c->fin_ring)))
        return launch_ring2(c, s, op, lo, hi, gap);
    // slab kernels read ghost planes refreshed from neighbours; one slab (2-D TMA grids keep
    // ghost rows for the two-substep kernels) wraps periodically like a plain grid
    const bool slab = c->ghost > 0 && c->slabs * c->loopback > 1;
    const bool lf = op.modeB == gbs::MODE_LF || op.modeB == gbs::tma::MODE_FEA;   // four level outputs
    gbs::tma::PairArgs a{};
    if (lf) {
        a.Av = field_ptr(c, s, op.Av.b, op.Av.f);
        a.Bu = field_ptr(c, s, op.Bu.b, op.Bu.f); a.Bv = field_ptr(c, s, op.Bv.b, op.Bv.f);
        a.Cu = field_ptr(c, s, op.Cu.b, op.Cu.f);
    } else {
        a.Av = a.Cu = nullptr;
        a.Bu = op.out_u ? op.out_u : field_ptr(c, s, op.Bu.b, 0);
        a.Bv = op.out_v ? op.out_v : field_ptr(c, s, op.Bu.b, 1);
    }
    a.Su = field_ptr(c, s, op.Su.b, op.Su.f);
    a.U = field_ptr(c, s, op.U.b, op.U.f);
    a.nx = (int)c->n[0]; a.ny = (int)c->n[1]; a.nz = (int)s.nz;
    a.plane = c->plane;
    const double sx = c->n[0] / c->len[0], sy = c->n[1] / c->len[1], sz = c->n[2] / c->len[2];
    a.sx2 = sx * sx; a.sy2 = sy * sy; a.sz2 = sz * sz;
    a.cfA = op.cfA; a.cfB = op.cfB; a.wh = op.wh;
    a.nonfinite = op.flag ? c->d_flag : nullptr;
    a.zlo = (int)lo; a.zhi = (int)hi;
    // planes per CTA: each CTA primes 2r planes and fills its pipeline once, so longer chunks
    // save a little (256 vs 128: +0.4% on C5 at 27.7 waves of CTAs) -- but only while the grid
    // keeps >= 8 waves (C4 at 256 planes: 3.5 waves, 5% slower than 128)
    const int64_t tiles = (c->n[0] / gbs::tma::TX) * (c->n[1] / gbs::tma::TY);
    const int zauto = tiles * ((hi - lo + 255) / 256) >= 8LL * c->sms ? 256 : 128;
    int zc = c->zchunk_pair_opt > 0 ? c->zchunk_pair_opt : c->zchunk_opt > 0 ? c->zchunk_opt : zauto;
    if (!lf && c->zchunk_fin_opt > 0) zc = c->zchunk_fin_opt;
    a.zchunk = (int)std::min<int64_t>(zc, hi - lo);
    a.band = tile_band(c, c->n[0] / gbs::tma::TX);
    a.hint = lf ? c->hint_opt : c->hint_fin_opt;
    dim3 grid((unsigned)((c->n[0] / gbs::tma::TX) * (c->n[1] / gbs::tma::TY)), 1u,
              (unsigned)((hi - lo + a.zchunk - 1) / a.zchunk));
    face_chunks(lo, hi, gap, a.zchunk, a.zskip, grid.z);
    gbs::tma::PairMaps m;
    m.su_a = s.tm[op.Su.b][op.Su.f][0]; m.su_b = s.tm[op.Su.b][op.Su.f][1]; m.su_c = s.tm[op.Su.b][op.Su.f][2];
    m.u_a = s.tm[op.U.b][op.U.f][0]; m.u_b = s.tm[op.U.b][op.U.f][1]; m.u_c = s.tm[op.U.b][op.U.f][2];
    m.sv = s.tm[op.Sv.b][op.Sv.f][0];
    m.pv = s.tm[op.Pv.b][op.Pv.f][0];
    m.acc_u = s.tm[op.Bu.b][0][0]; m.acc_v = s.tm[op.Bu.b][1][0];
    const int zbase = (int)c->ghost;
    cudaError_t e = cudaSuccess;
    gbs::tma::PeerPush pp;
    const gbs::tma::PeerPush* peer = make_peer(c, s, lf ? op.Bu : Slot{op.Bu.b, 0}, lf ? op.Cu : Slot{-1, 0}, pp);
#define PR(RR, SL)                                                                                          \
    switch (op.modeB) {                                                                                     \
        case gbs::MODE_LF: e = launch_pair_tma<RR, gbs::MODE_LF, SL>(m, a, zbase, grid, c->stream, peer); break;     \
        case gbs::tma::MODE_FEA: e = launch_pair_tma<RR, gbs::tma::MODE_FEA, SL>(m, a, zbase, grid, c->stream, peer); break; \
        case gbs::MODE_FIN0: e = launch_pair_tma<RR, gbs::MODE_FIN0, SL>(m, a, zbase, grid, c->stream, peer); break; \
        default: e = launch_pair_tma<RR, gbs::MODE_FINACC, SL>(m, a, zbase, grid, c->stream, peer); break;           \
    }
    if (c->R == 2) { if (slab) { PR(2, true) } else { PR(2, false) } }
    else { if (slab) { PR(4, true) } else { PR(4, false) } }
#undef PR
    if (e != cudaSuccess) return fail(c, GBS_E_CUDA, "pair kernel setup: %s", cudaGetErrorString(e));
    c->launches++;
    e = cudaGetLastError();
    if (e != cudaSuccess) return fail(c, GBS_E_CUDA, "kernel launch failed: %s", cudaGetErrorString(e));
    return GBS_OK;
}

// ---------------------------------------------------------------------------
// single-stencil-field 3-D kernel (gbs_wave3d_half.cuh): one half of a leap-frog pair,
// or the forward-Euler substep, over the planes [lo, hi) of slab s
// ---------------------------------------------------------------------------
template <int R, int KIND, bool SLAB, int TYH, int RPT>
static cudaError_t launch_half_tma(const gbs::tma::HalfMaps& m, const gbs::tma::HalfArgs& a, int zbase, dim3 grid,
                                   cudaStream_t st) {
    constexpr int D = TYH == gbs::tma::TY ? 4 : 3;
    using L = gbs::tma::HalfLayout<R, TYH, D>;
    auto k = gbs::tma::wave3d_half_tma<R, KIND, SLAB, TYH, RPT, D>;
    cudaError_t e = ensure_smem(reinterpret_cast<const void*>(k), L::bytes);
    if (e != cudaSuccess) return e;
    k<<<grid, dim3(32, TYH / RPT), L::bytes, st>>>(m, a, zbase);
    return cudaSuccess;
}

bool half_eligible(const gbs_ctx* c) {
    return c->pde == GBS_WAVE3D && c->use_half && c->tma_grid && !c->peer_on;
}

int launch_half(gbs_ctx* c, Slab& s, const HalfOperands& op, int64_t lo, int64_t hi, int64_t gap) {
    const bool slab = c->ghost > 0 && c->slabs * c->loopback > 1;
    const bool tall = c->n[1] % gbs::tma::TYH_TALL == 0 && c->half_tall;
    const int TYH = tall ? gbs::tma::TYH_TALL : gbs::tma::TY;
    const int rpt = tall && c->half_rpt == 4 ? 4 : 2;
    gbs::tma::HalfArgs a{};
    a.X = field_ptr(c, s, op.X.b, op.X.f);
    a.P = field_ptr(c, s, op.P.b, op.P.f);
    a.O1 = field_ptr(c, s, op.O1.b, op.O1.f);
    a.O2 = field_ptr(c, s, op.O2.b, op.O2.f);
    a.O3 = op.kind == gbs::tma::HALF_FE ? field_ptr(c, s, op.O3.b, op.O3.f) : nullptr;
    a.nx = (int)c->n[0]; a.ny = (int)c->n[1]; a.nz = (int)s.nz;
    a.plane = c->plane;
    const double sx = c->n[0] / c->len[0], sy = c->n[1] / c->len[1], sz = c->n[2] / c->len[2];
    a.sx2 = sx * sx; a.sy2 = sy * sy; a.sz2 = sz * sz;
    a.c1 = op.c1; a.c2 = op.c2;
    a.zlo = (int)lo; a.zhi = (int)hi;
    const int64_t tiles = (c->n[0] / gbs::tma::TX) * (c->n[1] / TYH);
    const int zauto = tiles * ((hi - lo + 255) / 256) >= 8LL * c->sms ? 256 : 128;
    const int zc = c->zchunk_pair_opt > 0 ? c->zchunk_pair_opt : c->zchunk_opt > 0 ? c->zchunk_opt : zauto;
    a.zchunk = (int)std::min<int64_t>(zc, hi - lo);
    a.band = tile_band(c, c->n[0] / gbs::tma::TX);
    a.hint = c->hint_half_opt;
    dim3 grid((unsigned)tiles, 1u, (unsigned)((hi - lo + a.zchunk - 1) / a.zchunk));
    face_chunks(lo, hi, gap, a.zchunk, a.zskip, grid.z);
    gbs::tma::HalfMaps m;
    m.x_a = s.tm[op.X.b][op.X.f][tall ? 3 : 0];
    m.x_b = s.tm[op.X.b][op.X.f][1];
    m.x_c = s.tm[op.X.b][op.X.f][tall ? 4 : 2];
    m.p = s.tm[op.P.b][op.P.f][tall ? 3 : 0];
    const int zbase = (int)c->ghost;
    cudaError_t e = cudaSuccess;
#define HL(RR, SL)                                                                                                   \
    if (op.kind == gbs::tma::HALF_FE) {                                                                              \
        if (!tall) e = launch_half_tma<RR, gbs::tma::HALF_FE, SL, gbs::tma::TY, 2>(m, a, zbase, grid, c->stream);     \
        else if (rpt == 4) e = launch_half_tma<RR, gbs::tma::HALF_FE, SL, gbs::tma::TYH_TALL, 4>(m, a, zbase, grid, c->stream); \
        else e = launch_half_tma<RR, gbs::tma::HALF_FE, SL, gbs::tma::TYH_TALL, 2>(m, a, zbase, grid, c->stream);    \
    } else {                                                                                                         \
        if (!tall) e = launch_half_tma<RR, gbs::tma::HALF_LF, SL, gbs::tma::TY, 2>(m, a, zbase, grid, c->stream);     \
        else if (rpt == 4) e = launch_half_tma<RR, gbs::tma::HALF_LF, SL, gbs::tma::TYH_TALL, 4>(m, a, zbase, grid, c->stream); \
        else e = launch_half_tma<RR, gbs::tma::HALF_LF, SL, gbs::tma::TYH_TALL, 2>(m, a, zbase, grid, c->stream);    \
    }
    if (c->R == 2) { if (slab) { HL(2, true) } else { HL(2, false) } }
    else { if (slab) { HL(4, true) } else { HL(4, false) } }
#undef HL
    if (e != cudaSuccess) return fail(c, GBS_E_CUDA, "half kernel setup: %s", cudaGetErrorString(e));
    c->launches++;
    e = cudaGetLastError();
    if (e != cudaSuccess) return fail(c, GBS_E_CUDA, "kernel launch failed: %s", cudaGetErrorString(e));
    return GBS_OK;
}

int launch_ghost_fill(gbs_ctx* c, const std::vector<std::pair<int, unsigned>>& halos) {
    gbs::GhostFillArgs a{};
    Slab& s = c->slab[0];
    for (auto& h : halos)
        for (int f = 0; f < c->F; ++f)
            if ((h.second >> f) & 1u) {
                if (a.nf == 6) return fail(c, GBS_E_INVAL, "ghost_fill: more than 6 fields");
                a.f[a.nf++] = field_ptr(c, s, h.first, f);
            }
    if (!a.nf) return GBS_OK;
    a.n = s.nz; a.g = c->ghost; a.plane = c->plane;
    const int64_t per = a.g * a.plane;
    dim3 grid((unsigned)std::min<int64_t>((per + 255) / 256, 4 * c->sms), (unsigned)a.nf);
    gbs::ghost_fill<<<grid, 256, 0, c->stream>>>(a);
    c->launches++;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(c, GBS_E_CUDA, "ghost fill launch failed: %s", cudaGetErrorString(e));
    return GBS_OK;
}

// ---------------------------------------------------------------------------
// 2-D acoustics, two leap-frog substeps per pass (gbs_acoustic2d_pair.cuh): the
// chain-U kernel then the chain-P kernel over the rows [lo, hi) of slab s
// ---------------------------------------------------------------------------
template <int R>
static cudaError_t launch_ac2d_chains(const gbs::tma::Ac2PairMaps& m, const gbs::tma::Ac2PairArgs& a, int ybase,
                                      dim3 grid, cudaStream_t st) {
    using LU = gbs::tma::ChainULayout<R>;
    using LP = gbs::tma::ChainPLayout<R>;
    cudaError_t e = ensure_smem(reinterpret_cast<const void*>(gbs::tma::acoustic2d_chainU_tma<R>), LU::bytes);
    if (e == cudaSuccess) e = ensure_smem(reinterpret_cast<const void*>(gbs::tma::acoustic2d_chainP_tma<R>), LP::bytes);
    if (e != cudaSuccess) return e;
    const dim3 block(32, gbs::tma::AC2_NW + 1);
    gbs::tma::acoustic2d_chainU_tma<R><<<grid, block, LU::bytes, st>>>(m, a, ybase);
    gbs::tma::acoustic2d_chainP_tma<R><<<grid, block, LP::bytes, st>>>(m, a, ybase);
    return cudaSuccess;
}

int launch_ac2d_pair(gbs_ctx* c, Slab& s, int P, int S, int Aout, int Bout, double cfA, double cfB, int64_t lo,
                     int64_t hi, int64_t gap) {
    gbs::tma::Ac2PairArgs a{};
    for (int f = 0; f < 3; ++f) {
        a.A[f] = field_ptr(c, s, Aout, f);
        a.B[f] = field_ptr(c, s, Bout, f);
    }
    a.nx = (int)c->n[0]; a.ny = (int)s.nz;
    a.ylo = (int)lo; a.yhi = (int)hi;
    a.sx = c->n[0] / c->len[0]; a.sy = c->n[1] / c->len[1];
    a.cfA = cfA; a.cfB = cfB;
    const int64_t xt = c->n[0] / gbs::tma::TX;
    a.ychunk = ac2d_ychunk(xt, hi - lo, c->zchunk_opt, c->sms, gbs::tma::AC2_BH);
    dim3 grid((unsigned)xt, (unsigned)((hi - lo + a.ychunk - 1) / a.ychunk));
    face_chunks(lo, hi, gap, a.ychunk, a.yskip, grid.y);
    gbs::tma::Ac2PairMaps m;
    static const int pick[6] = {3, 4, 5, 6, 7, 8};      // Ac2PairMaps box order -> tm shape index
    for (int f = 0; f < 3; ++f)
        for (int k = 0; k < 6; ++k) {
            m.s[f][k] = s.tm[S][f][pick[k]];
            m.p[f][k] = s.tm[P][f][pick[k]];
        }
    const int ybase = (int)c->ghost;
    cudaError_t e = c->R == 2 ? launch_ac2d_chains<2>(m, a, ybase, grid, c->stream)
                              : launch_ac2d_chains<4>(m, a, ybase, grid, c->stream);
    if (e != cudaSuccess) return fail(c, GBS_E_CUDA, "2-D pair kernel setup: %s", cudaGetErrorString(e));
    c->launches += 2;
    e = cudaGetLastError();
    if (e != cudaSuccess) return fail(c, GBS_E_CUDA, "kernel launch failed: %s", cudaGetErrorString(e));
    return GBS_OK;
}

// ---------------------------------------------------------------------------
// small 1-D grids: the whole run in one cluster launch (K6)
// ---------------------------------------------------------------------------

bool persistent_path(const gbs_ctx* c) {
    const int m = (int)c->my_seq.size();
    return c->use_persistent && c->pde == GBS_ADV1D && c->world == 1 && c->loopback == 1 && m >= 1 &&
           m <= 16 && c->n[0] <= (c->order == 0 ? kSpectralMaxN : kClusterMaxN);
}

// ---------------------------------------------------------------------------
// spectral derivative beyond the cluster kernel: per substep D2Z, multiply by
// i 2 pi k / (L N) (Nyquist dropped), Z2D -- the derivative of the trigonometric
// interpolant (the oracle's definition, R20) -- then the
// pointwise FE / LF / final update
// ---------------------------------------------------------------------------
int spectral_setup(gbs_ctx* c) {
    if (c->order != 0 || c->fft_fwd >= 0) return GBS_OK;
    auto& F = cufft::api();
    if (!F.ok) return fail(c, GBS_E_UNSUPPORTED, "libcufft.so.11 not found (spectral derivative, N > %d)",
                           kSpectralMaxN);
    const int n = (int)c->n[0];
    CU(c, cudaMalloc(&c->fft_buf, sizeof(double) * (size_t)(2 * (n / 2 + 1) + n)));
    int r = F.Plan1d(&c->fft_fwd, n, cufft::D2Z, 1);
    if (!r) r = F.Plan1d(&c->fft_inv, n, cufft::Z2D, 1);
    if (!r) r = F.SetStream(c->fft_fwd, c->stream);
    if (!r) r = F.SetStream(c->fft_inv, c->stream);
    if (r) return fail(c, GBS_E_CUDA, "cuFFT plan setup failed (%d)", r);
    return GBS_OK;
}

void spectral_release(gbs_ctx* c) {
    auto& F = cufft::api();
    if (F.ok) {
        if (c->fft_fwd >= 0) F.Destroy(c->fft_fwd);
        if (c->fft_inv >= 0) F.Destroy(c->fft_inv);
    }
    c->fft_fwd = c->fft_inv = -1;
    if (c->fft_buf) cudaFree(c->fft_buf);
    c->fft_buf = nullptr;
}

static int launch_spectral_step(gbs_ctx* c, const gbs::Adv1DArgs& a, int mode) {
    auto& F = cufft::api();
    const int n = a.nx;
    double2* spec = reinterpret_cast<double2*>(c->fft_buf);
    double* du = c->fft_buf + 2 * (n / 2 + 1);
    int r = F.ExecD2Z(c->fft_fwd, const_cast<double*>(a.S), spec);
    if (r) return fail(c, GBS_E_CUDA, "cufftExecD2Z failed (%d)", r);
    const double s = 2.0 * 3.14159265358979323846 / (c->len[0] * (double)n);
    gbs::spectral_ik<<<(unsigned)((n / 2 + 1 + 255) / 256), 256, 0, c->stream>>>(spec, n, s);
    r = F.ExecZ2D(c->fft_inv, spec, du);
    if (r) return fail(c, GBS_E_CUDA, "cufftExecZ2D failed (%d)", r);
    const unsigned g = (unsigned)((n + 255) / 256);
    switch (mode) {
        case gbs::MODE_FE: gbs::adv1d_spectral_update<gbs::MODE_FE><<<g, 256, 0, c->stream>>>(a, du); break;
        case gbs::MODE_LF: gbs::adv1d_spectral_update<gbs::MODE_LF><<<g, 256, 0, c->stream>>>(a, du); break;
        case gbs::MODE_FIN0: gbs::adv1d_spectral_update<gbs::MODE_FIN0><<<g, 256, 0, c->stream>>>(a, du); break;
        default: gbs::adv1d_spectral_update<gbs::MODE_FINACC><<<g, 256, 0, c->stream>>>(a, du); break;
    }
    c->launches += 2;                                  // ours; cuFFT's own kernels not counted
    return GBS_OK;
}

int launch_cluster_run(gbs_ctx* c, int64_t macro_steps, double H) {
    const int m = (int)c->my_seq.size();
    if (!c->d_nk) {
        std::vector<int> nk;
        std::vector<double> wh;
        for (int k : c->my_seq) { nk.push_back(c->nk_all[k]); wh.push_back(0.5 * c->wk_all[k]); }
        CU(c, cudaMalloc(&c->d_nk, sizeof(int) * m));
        CU(c, cudaMalloc(&c->d_wh, sizeof(double) * m));
        CU(c, cudaMemcpyAsync(c->d_nk, nk.data(), sizeof(int) * m, cudaMemcpyHostToDevice, c->stream));
        CU(c, cudaMemcpyAsync(c->d_wh, wh.data(), sizeof(double) * m, cudaMemcpyHostToDevice, c->stream));
    }
    gbs::Adv1DClusterArgs a;
    a.Y = field_ptr(c, c->slab[0], c->yb, 0);
    a.nx = (int)c->n[0];
    a.sx = c->n[0] / c->len[0];
    a.H = H;
    a.macro_steps = macro_steps;
    a.nk = c->d_nk;
    a.wh = c->d_wh;
    a.nonfinite = c->d_flag;
    const bool spectral = c->order == 0;
    const size_t smem = sizeof(double) * (4 * (size_t)a.nx + (spectral ? (size_t)a.nx / 2 : 0));
    if (spectral && !c->d_alpha) {
        // alpha_j = pi (-1)^{j+1} cot(j pi / N) / N, j = 1 .. N/2 - 1 (gbs_adv1d_cluster.cuh)
        const int64_t N = c->n[0];
        std::vector<double> al((size_t)(N / 2 - 1));
        for (int64_t j = 1; j <= N / 2 - 1; ++j)
            al[(size_t)(j - 1)] = (j % 2 ? 1.0 : -1.0) * M_PI / std::tan((double)j * M_PI / (double)N) / (double)N;
        CU(c, cudaMalloc(&c->d_alpha, sizeof(double) * al.size() + 8));
        CU(c, cudaMemcpyAsync(c->d_alpha, al.data(), sizeof(double) * al.size(), cudaMemcpyHostToDevice,
                              c->stream));
    }
    int rc;
    cudaEvent_t end = nullptr;
    if (spectral) {
        auto kern = gbs::adv1d_cluster_run_spectral;
        CU(c, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        if (m > 8) CU(c, cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)m);
        cfg.blockDim = dim3(256);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = c->stream;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = (unsigned)m;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        const double* alpha = c->d_alpha;
        if (c->time_kernels && (rc = timed_begin(c, 5, &end))) return rc;
        CU(c, cudaLaunchKernelEx(&cfg, kern, a, alpha));
        if (end) CU(c, cudaEventRecord(end, c->stream));
        c->launches++;
        return GBS_OK;
    }
    void (*kern)(const gbs::Adv1DClusterArgs) =
        c->R == 2 ? gbs::adv1d_cluster_run<2> : gbs::adv1d_cluster_run<4>;
    CU(c, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    if (m > 8) CU(c, cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)m);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = c->stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)m;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (c->time_kernels && (rc = timed_begin(c, 5, &end))) return rc;
    CU(c, cudaLaunchKernelEx(&cfg, kern, a));
    if (end) CU(c, cudaEventRecord(end, c->stream));
    c->launches++;
    return GBS_OK;
}

// gbs_api.cu -- the C ABI (include/gbs.h): validation, planning, device
// memory, the per-macro-step schedule (optionally a CUDA graph), the
// slab halo exchange and the cross-GPU combine over NCCL.
//
// The schedule of one macro step (Eq. (1), lines 85-98, and the
// combination at lines 109-115, 221-225), per local slab:
//   for each sequence k of this rank's group, ascending n_k, h = H / n_k:
//     FE       B  = Y + h f(Y)                        (kernel MODE_FE)
//     LF_1     C  = Y + 2h f(B)                       (MODE_LF, fresh buffer)
//     LF_i     prev = prev + 2h f(cur), swap           (MODE_LF in place), i = 2..n_k-1
//     final    ACC (+)= w_k/2 (prev + cur + h f(cur))  (MODE_FIN0 / MODE_FINACC)
//   [multi-GPU] ACC <- sum over sequence groups        (ncclAllReduce, fp64 sum)
//   swap(Y, ACC)
// Before every stencil launch on a slabbed grid the source level's ghost
// planes are refreshed from the neighbouring slabs (cudaMemcpyAsync between
// local slabs in loopback mode, ncclSend/ncclRecv between ranks).
#include "gbs.h"
#include "gbs_kernels.cuh"
#include "gbs_wave3d_tma.cuh"
#include "gbs_wave3d_pair.cuh"
#include "gbs_acoustic2d_tma.cuh"
#include "gbs_adv1d_cluster.cuh"

#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

// ---------------------------------------------------------------------------
// NCCL, resolved at run time from the process (torch's libnccl.so.2) so the
// library loads on machines without NCCL and never links a second copy.
// ---------------------------------------------------------------------------
namespace nccl {
typedef struct ncclComm* comm_t;
typedef struct { char internal[128]; } uid_t;
enum { ncclSuccess = 0 };
enum { ncclFloat64 = 8 };
enum { ncclSum = 0 };
typedef int (*GetUniqueId_t)(uid_t*);
typedef int (*CommInitRank_t)(comm_t*, int, uid_t, int);
typedef int (*CommSplit_t)(comm_t, int, int, comm_t*, void*);
typedef int (*CommDestroy_t)(comm_t);
typedef int (*AllReduce_t)(const void*, void*, size_t, int, int, comm_t, cudaStream_t);
typedef int (*AllGather_t)(const void*, void*, size_t, int, comm_t, cudaStream_t);
typedef int (*Send_t)(const void*, size_t, int, int, comm_t, cudaStream_t);
typedef int (*Recv_t)(void*, size_t, int, int, comm_t, cudaStream_t);
typedef int (*Group_t)(void);
typedef const char* (*GetErrorString_t)(int);
struct Api {
    bool ok = false;
    GetUniqueId_t GetUniqueId; CommInitRank_t CommInitRank; CommSplit_t CommSplit;
    CommDestroy_t CommDestroy; AllReduce_t AllReduce; AllGather_t AllGather;
    Send_t Send; Recv_t Recv; Group_t GroupStart, GroupEnd; GetErrorString_t GetErrorString;
};
static Api& api() {
    static Api a;
    static bool tried = false;
    if (tried) return a;
    tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return a;
#define NCCL_SYM(name) a.name = (decltype(a.name))dlsym(h, "nccl" #name); if (!a.name) return a;
    NCCL_SYM(GetUniqueId) NCCL_SYM(CommInitRank) NCCL_SYM(CommSplit) NCCL_SYM(CommDestroy)
    NCCL_SYM(AllReduce) NCCL_SYM(AllGather) NCCL_SYM(Send) NCCL_SYM(Recv)
    NCCL_SYM(GroupStart) NCCL_SYM(GroupEnd) NCCL_SYM(GetErrorString)
#undef NCCL_SYM
    a.ok = true;
    return a;
}
}  // namespace nccl

// ---------------------------------------------------------------------------
struct Slab {
    int64_t z0 = 0, nz = 0;           // interior planes [z0, z0 + nz) of the slowest axis
    double* buf[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};   // Y, ACC, L0..L3 (+ ghosts)
    bool tma_ok = false;              // tensor maps below are valid (TMA kernels eligible)
    CUtensorMap tm[6][3][3];          // [buffer][field][box shape A/B/C] (TMA kernels)
};

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

static constexpr int kClusterMaxN = 7000;     // 4 nx doubles of shared memory per CTA
static constexpr int kSpectralMaxN = 6400;    // 4.5 nx doubles (state, levels, weights)

struct KernelTimer {
    std::vector<cudaEvent_t> ev;      // pairs
    std::vector<int> cls;
    size_t used = 0;
    double total_ms[6] = {0, 0, 0, 0, 0, 0};
    int64_t launches[6] = {0, 0, 0, 0, 0, 0};
};

struct gbs_ctx {
    // problem
    int pde = 0, ndim = 0, F = 0, order = 0, R = 0;
    int64_t n[3] = {1, 1, 1};
    double len[3] = {1, 1, 1};
    int64_t plane = 0;                // points per plane of the slowest axis
    int64_t nslow = 0;                // extent of the slowest axis
    int64_t points = 0;
    // scheme (ascending n_k)
    std::vector<int> nk_all;
    std::vector<double> wk_all;
    std::vector<int> my_seq;          // indices into nk_all run by this rank
    // distribution
    int rank = 0, world = 1, device = 0, groups = 1, slabs = 1, my_group = 0, my_slab = 0;
    int loopback = 1;                 // local slabs on this GPU
    nccl::comm_t comm_world = nullptr, comm_slab = nullptr, comm_group = nullptr;
    // memory
    std::vector<Slab> slab;
    int64_t ghost = 0;                // ghost planes per side (R when slabbed)
    int64_t field_stride = 0;         // doubles per field incl. ghosts
    int yb = 0;                       // which of buf[0]/buf[1] is Y
    int* d_flag = nullptr;
    double* d_gather = nullptr;       // multi-GPU read_state staging
    // execution
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    bool have_state = false;
    bool use_graph = true;
    bool time_kernels = false;
    bool use_bulk = true;             // bulk-copy (TMA engine) pipelined kernels where eligible
    bool use_persistent = true;       // one cluster launch per gbs_advance for small 1-D grids
    double* d_alpha = nullptr;        // spectral derivative weights (order 0)
    // asynchronous slab IO (gbs_write_slab_async / gbs_read_slab_async): per local slab a
    // staging buffer for the incoming and for the outgoing state, own copy streams
    std::vector<double*> in_buf, out_buf;
    cudaStream_t h2d = nullptr, d2h = nullptr;
    cudaEvent_t ev_in_ready = nullptr, ev_in_free = nullptr, ev_out_ready = nullptr, ev_out_free = nullptr;
    bool pending_in = false;
    // halo exchange overlapped with the interior planes (slabbed layouts)
    bool use_overlap = true;
    cudaStream_t cstream = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    int* d_nk = nullptr;              // step counts / half weights for the cluster kernel
    double* d_wh = nullptr;
    bool use_fuse = true;             // two-substep (temporally blocked) kernels where eligible
                                      // (bit-exact)
    bool tma_grid = false;            // grid is a multiple of the TMA tile (wave3d)
    int nbuf = 4;                     // state buffers per slab: Y, ACC + 2 or 4 level buffers
    int zchunk_opt = 0;
    int sms = 148;                    // streaming multiprocessors of the device
    cudaGraphExec_t gexec[2] = {nullptr, nullptr};
    double graph_H = -1.0;
    int64_t macro_done = 0;
    int64_t launches = 0;
    int64_t launches_per_macro = 0;
    double t = 0.0;
    KernelTimer timer;
    std::string err;
};

static thread_local std::string g_err;

static int fail(gbs_ctx* c, int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    if (c) c->err = buf;
    g_err = buf;
    return code;
}

#define CU(c, call)                                                                      \
    do {                                                                                 \
        cudaError_t e_ = (call);                                                         \
        if (e_ != cudaSuccess)                                                           \
            return fail(c, GBS_E_CUDA, "%s failed: %s", #call, cudaGetErrorString(e_)); \
    } while (0)

#define NC(c, call)                                                                         \
    do {                                                                                    \
        int r_ = (call);                                                                    \
        if (r_ != nccl::ncclSuccess)                                                        \
            return fail(c, GBS_E_NCCL, "%s failed: %s", #call, nccl::api().GetErrorString(r_)); \
    } while (0)

// ---------------------------------------------------------------------------
// planning
// ---------------------------------------------------------------------------
// Partition sequence indices into g groups with balanced sum(n_k + 1): longest
// processing time first, then pairwise moves/swaps while the maximum drops.
static std::vector<std::vector<int>> partition(const std::vector<int>& nk, int g) {
    int m = (int)nk.size();
    std::vector<int> order(m);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return nk[a] > nk[b]; });
    std::vector<std::vector<int>> grp(g);
    std::vector<int64_t> load(g, 0);
    for (int i : order) {
        int best = (int)(std::min_element(load.begin(), load.end()) - load.begin());
        grp[best].push_back(i);
        load[best] += nk[i] + 1;
    }
    bool improved = true;
    while (improved) {
        improved = false;
        int hi = (int)(std::max_element(load.begin(), load.end()) - load.begin());
        for (int o = 0; o < g && !improved; ++o) {
            if (o == hi) continue;
            for (size_t a = 0; a < grp[hi].size() && !improved; ++a) {
                int ia = grp[hi][a];
                // move
                int64_t nh = load[hi] - (nk[ia] + 1), no = load[o] + (nk[ia] + 1);
                if (std::max(nh, no) < load[hi]) {
                    grp[o].push_back(ia); grp[hi].erase(grp[hi].begin() + a);
                    load[hi] = nh; load[o] = no; improved = true; break;
                }
                for (size_t b = 0; b < grp[o].size(); ++b) {
                    int ib = grp[o][b];
                    int64_t d = (int64_t)nk[ia] - nk[ib];
                    if (d > 0 && std::max(load[hi] - d, load[o] + d) < load[hi]) {
                        std::swap(grp[hi][a], grp[o][b]);
                        load[hi] -= d; load[o] += d; improved = true; break;
                    }
                }
            }
        }
    }
    for (auto& v : grp) std::sort(v.begin(), v.end(), [&](int a, int b) { return nk[a] < nk[b]; });
    return grp;
}

static int64_t crit_path(const std::vector<int>& nk, int g) {
    auto grp = partition(nk, g);
    int64_t mx = 0;
    for (auto& v : grp) {
        int64_t s = 0;
        for (int i : v) s += nk[i] + 1;
        mx = std::max(mx, s);
    }
    return mx;
}

// Choose g sequence groups x s slabs (g * s = world) minimising the modelled
// per-GPU time of one macro step: stencil bytes at HBM
// bandwidth + per-substep halo bytes at NVLink bandwidth + allreduce bytes.
static void plan(gbs_ctx* c, int want_groups) {
    const int W = c->world;
    double best = 1e300;
    int bg = 1;
    for (int g = 1; g <= W; ++g) {
        if (W % g) continue;
        int s = W / g;
        if (want_groups > 0 && g != want_groups) continue;
        if (g > (int)c->nk_all.size()) continue;
        if (s > 1 && (c->ndim == 1 || c->nslow % s || c->nslow / s < c->R)) continue;
        double crit = (double)crit_path(c->nk_all, g);
        double pts = (double)c->points / s;
        double t_comp = crit * pts * 24.0 * c->F / 6.5e12;
        double halo_fields = c->pde == GBS_WAVE3D ? 1.0 : 2.0;
        double t_halo = s > 1 ? crit * (2.0 * c->R * c->plane * 8.0 * halo_fields / 7.7e11 + 2e-5) : 0.0;
        // the exchange overlaps the interior planes; only what exceeds them is exposed
        const double nzs = (double)c->nslow / s;
        if (s > 1 && c->use_overlap && nzs >= 3.0 * 16.0)
            t_halo = std::max(0.0, t_halo - t_comp * (nzs - 2.0 * 16.0) / nzs);
        double state = pts * c->F * 8.0;
        double t_ar = g > 1 ? 2.0 * (g - 1) / g * state / 7.0e11 + 5e-5 : 0.0;
        double tot = t_comp + t_halo + t_ar;
        if (tot < best * (1 - 1e-9)) { best = tot; bg = g; }
    }
    c->groups = bg;
    c->slabs = W / bg;
}

// ---------------------------------------------------------------------------
// memory helpers
// ---------------------------------------------------------------------------
static inline double* field_ptr(gbs_ctx* c, Slab& s, int b, int f) {
    return s.buf[b] + (int64_t)f * c->field_stride + c->ghost * c->plane;
}

static int alloc_state(gbs_ctx* c) {
    int nloc = c->loopback;
    int64_t total_slabs = (int64_t)c->slabs * nloc;
    int64_t nzl = c->nslow / total_slabs;
    c->ghost = total_slabs > 1 ? c->R : 0;
    c->field_stride = (nzl + 2 * c->ghost) * c->plane;
    // the TMA (and two-substep) kernels need the grid to be a multiple of their tile so
    // halo boxes never cross the wrap; the two-substep kernels need 4 level buffers
    // (2-D acoustics: x a multiple of the tile width, each slab's rows a multiple of its height)
    c->tma_grid = (c->pde == GBS_WAVE3D && c->n[0] % gbs::tma::TX == 0 && c->n[1] % gbs::tma::TY == 0) ||
                  (c->pde == GBS_ACOUSTIC2D && c->n[0] % gbs::tma::TX == 0 && nzl % gbs::tma::TY == 0);
    c->nbuf = (c->tma_grid && c->pde == GBS_WAVE3D) ? 6 : 4;
    c->slab.resize(nloc);
    for (int v = 0; v < nloc; ++v) {
        Slab& s = c->slab[v];
        int64_t gidx = (int64_t)c->my_slab * nloc + v;
        s.z0 = gidx * nzl;
        s.nz = nzl;
        for (int b = 0; b < c->nbuf; ++b) {
            size_t bytes = sizeof(double) * (size_t)c->F * (size_t)c->field_stride;
            if (cudaMalloc(&s.buf[b], bytes) != cudaSuccess)
                return fail(c, GBS_E_NOMEM, "cudaMalloc of %zu bytes failed", bytes);
            CU(c, cudaMemsetAsync(s.buf[b], 0, bytes, c->stream));
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
                }
            s.tma_ok = ok;
        }
    }
    CU(c, cudaMalloc(&c->d_flag, sizeof(int)));
    CU(c, cudaMemsetAsync(c->d_flag, 0, sizeof(int), c->stream));
    return GBS_OK;
}

static void free_state(gbs_ctx* c) {
    for (auto& s : c->slab)
        for (int b = 0; b < 6; ++b)
            if (s.buf[b]) { cudaFree(s.buf[b]); s.buf[b] = nullptr; }
    c->slab.clear();
}

// ---------------------------------------------------------------------------
// kernel dispatch
// ---------------------------------------------------------------------------
struct Slot { int b, f; };   // one field of one state buffer
struct StepOperands {
    int S, P, O;          // buffer indices of the current level, previous level, output
    int mode;
    double cf, wh;
    bool flag;
    Slot xu = {-1, 0};    // FE only (TMA kernel): also write u_2 = S_u + cf2 v_1 here
    double cf2 = 0.0;
};

template <int R, int MODE, bool SLAB>
static void launch_wave3d(const gbs::Wave3DArgs& a, dim3 grid, bool vx2, cudaStream_t st) {
    if (vx2) gbs::wave3d_step<R, MODE, 2, 16, SLAB><<<grid, dim3(32, 16), 0, st>>>(a);
    else gbs::wave3d_step<R, MODE, 1, 16, SLAB><<<grid, dim3(32, 16), 0, st>>>(a);
}
template <int R, int MODE, bool SLAB>
static cudaError_t launch_wave3d_tma(const gbs::tma::Maps& m, const gbs::Wave3DArgs& a, int zbase, dim3 grid,
                                     cudaStream_t st) {
    using L = gbs::tma::Layout<R, MODE>;
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(gbs::tma::wave3d_step_tma<R, MODE, SLAB>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::bytes);
        if (e != cudaSuccess) return e;
        configured = true;
    }
    gbs::tma::wave3d_step_tma<R, MODE, SLAB><<<grid, dim3(32, gbs::tma::TY + 1), L::bytes, st>>>(m, a, zbase);
    return cudaSuccess;
}
template <int R, int MODEB, bool SLAB>
static cudaError_t launch_pair_tma(const gbs::tma::PairMaps& m, const gbs::tma::PairArgs& a, int zbase, dim3 grid,
                                   cudaStream_t st) {
    using L = gbs::tma::PairLayout<R, MODEB>;
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(gbs::tma::wave3d_pair_tma<R, MODEB, SLAB>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::bytes);
        if (e != cudaSuccess) return e;
        configured = true;
    }
    gbs::tma::wave3d_pair_tma<R, MODEB, SLAB><<<grid, dim3(32, gbs::tma::TY / 2), L::bytes, st>>>(m, a, zbase);
    return cudaSuccess;
}
template <int R, int MODE, bool SLAB>
static cudaError_t launch_ac2d_tma(const gbs::tma::AcMaps& m, const gbs::Acoustic2DArgs& a, int ybase, dim3 grid,
                                   cudaStream_t st) {
    using L = gbs::tma::AcLayout<R, MODE>;
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(gbs::tma::acoustic2d_step_tma<R, MODE, SLAB>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::bytes);
        if (e != cudaSuccess) return e;
        configured = true;
    }
    gbs::tma::acoustic2d_step_tma<R, MODE, SLAB><<<grid, dim3(32, gbs::tma::TY + 1), L::bytes, st>>>(m, a, ybase);
    return cudaSuccess;
}
// rows per CTA of the 2-D TMA kernel: a multiple of the tile height minimising
// (waves of one-CTA-per-SM) x (rows + ~2 tiles of pipeline fill)
static int ac2d_ychunk(int64_t xtiles, int64_t ny, int opt, int sms) {
    const int T = gbs::tma::TY;
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
static int launch_step(gbs_ctx* c, Slab& s, const StepOperands& op, int64_t lo, int64_t hi) {
    const bool slab = c->ghost > 0;
    int* flag = op.flag ? c->d_flag : nullptr;
    if (c->pde == GBS_WAVE3D) {
        gbs::Wave3DArgs a;
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
            dim3 grid((unsigned)tx, (unsigned)ty, (unsigned)((hi - lo + a.zchunk - 1) / a.zchunk));
            gbs::tma::Maps m;
            m.su_a = s.tm[op.S][0][0]; m.su_b = s.tm[op.S][0][1]; m.su_c = s.tm[op.S][0][2];
            m.sv = s.tm[op.S][1][0];
            m.pu = s.tm[op.P][0][0]; m.pv = s.tm[op.P][1][0];
            m.au = s.tm[op.O][0][0]; m.av = s.tm[op.O][1][0];
            const int zbase = (int)c->ghost;
            cudaError_t e = cudaSuccess;
#define W3B(RR, SL)                                                                                   \
            switch (op.mode) {                                                                        \
                case gbs::MODE_FE: e = launch_wave3d_tma<RR, gbs::MODE_FE, SL>(m, a, zbase, grid, c->stream); break;     \
                case gbs::MODE_LF: e = launch_wave3d_tma<RR, gbs::MODE_LF, SL>(m, a, zbase, grid, c->stream); break;     \
                case gbs::MODE_FIN0: e = launch_wave3d_tma<RR, gbs::MODE_FIN0, SL>(m, a, zbase, grid, c->stream); break; \
                default: e = launch_wave3d_tma<RR, gbs::MODE_FINACC, SL>(m, a, zbase, grid, c->stream); break;           \
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
        gbs::Acoustic2DArgs a;
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

// Two consecutive substeps of one sequence in one launch (3-D wave, TMA grids),
// gbs_wave3d_pair.cuh.  Operands are field slots (buffer, field): the pair
// kernel reads P_v, S = (S_u, S_v) and U = u_{n+1}; LF writes Av = v_{n+1},
// (Bu, Bv) = y_{n+2} and Cu = u_{n+3}; FIN0/FINACC writes the accumulator
// buffer's two fields only.
struct PairOperands {
    Slot Pv, Su, Sv, U;
    Slot Av, Bu, Bv, Cu;          // LF outputs (Bu.b = the accumulator buffer for FIN)
    int modeB;
    double cfA, cfB, wh;
    bool flag;
};

static int launch_pair(gbs_ctx* c, Slab& s, const PairOperands& op, int64_t lo, int64_t hi) {
    const bool slab = c->ghost > 0;
    const bool lf = op.modeB == gbs::MODE_LF;
    gbs::tma::PairArgs a;
    if (lf) {
        a.Av = field_ptr(c, s, op.Av.b, op.Av.f);
        a.Bu = field_ptr(c, s, op.Bu.b, op.Bu.f); a.Bv = field_ptr(c, s, op.Bv.b, op.Bv.f);
        a.Cu = field_ptr(c, s, op.Cu.b, op.Cu.f);
    } else {
        a.Av = a.Cu = nullptr;
        a.Bu = field_ptr(c, s, op.Bu.b, 0); a.Bv = field_ptr(c, s, op.Bu.b, 1);
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
    a.zchunk = c->zchunk_opt > 0 ? (int)std::min<int64_t>(c->zchunk_opt, hi - lo) : (int)std::min<int64_t>(128, hi - lo);
    dim3 grid((unsigned)(c->n[0] / gbs::tma::TX), (unsigned)(c->n[1] / gbs::tma::TY),
              (unsigned)((hi - lo + a.zchunk - 1) / a.zchunk));
    gbs::tma::PairMaps m;
    m.su_a = s.tm[op.Su.b][op.Su.f][0]; m.su_b = s.tm[op.Su.b][op.Su.f][1]; m.su_c = s.tm[op.Su.b][op.Su.f][2];
    m.u_a = s.tm[op.U.b][op.U.f][0]; m.u_b = s.tm[op.U.b][op.U.f][1]; m.u_c = s.tm[op.U.b][op.U.f][2];
    m.sv = s.tm[op.Sv.b][op.Sv.f][0];
    m.pv = s.tm[op.Pv.b][op.Pv.f][0];
    m.acc_u = s.tm[op.Bu.b][0][0]; m.acc_v = s.tm[op.Bu.b][1][0];
    const int zbase = (int)c->ghost;
    cudaError_t e = cudaSuccess;
#define PR(RR, SL)                                                                                          \
    switch (op.modeB) {                                                                                     \
        case gbs::MODE_LF: e = launch_pair_tma<RR, gbs::MODE_LF, SL>(m, a, zbase, grid, c->stream); break;     \
        case gbs::MODE_FIN0: e = launch_pair_tma<RR, gbs::MODE_FIN0, SL>(m, a, zbase, grid, c->stream); break; \
        default: e = launch_pair_tma<RR, gbs::MODE_FINACC, SL>(m, a, zbase, grid, c->stream); break;           \
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
// The per-substep halo schedule of one slab (posted inside one NCCL group).
// Per field: send up (my top interior planes -> the upper neighbour's low
// ghosts), send down (my bottom interior planes -> the lower neighbour's high
// ghosts), receive from below (into my low ghosts), receive from above (into
// my high ghosts).  NCCL matches p2p operations per peer pair in posting order:
// slab a's k-th send to b is b's k-th receive from a.  With 2 slabs both
// neighbours are the same peer and the order send-up/send-down vs
// recv-low/recv-high pairs a's top planes with b's low ghosts -- as required.
// ---------------------------------------------------------------------------
static std::vector<gbs_halo_op> halo_schedule(int slabs, int my_slab, int64_t nz, int G, unsigned mask) {
    std::vector<gbs_halo_op> ops;
    if (slabs < 2) return ops;
    const int lo = (my_slab - 1 + slabs) % slabs, hi = (my_slab + 1) % slabs;
    for (int f = 0; f < 32; ++f) {
        if (!(mask & (1u << f))) continue;
        ops.push_back({0, hi, f, 0, nz - G, G});      // send up
        ops.push_back({0, lo, f, 0, 0, G});           // send down
        ops.push_back({1, lo, f, 0, -G, G});          // receive from below
        ops.push_back({1, hi, f, 0, nz, G});          // receive from above
    }
    return ops;
}

// ---------------------------------------------------------------------------
// halo exchange of buffer b's fields in `mask` (bit f = field f; 0 = the fields
// whose stencil crosses the slab axis) -- ghost planes along the slowest axis
// ---------------------------------------------------------------------------
static int exchange_halo(gbs_ctx* c, int b, unsigned mask = 0, cudaStream_t st = nullptr) {
    if (!st) st = c->stream;
    if (c->ghost == 0) return GBS_OK;
    const int64_t G = c->ghost, P = c->plane;
    const size_t cnt = (size_t)(G * P);
    std::vector<int> fields;
    if (mask) {
        for (int f = 0; f < c->F; ++f)
            if (mask & (1u << f)) fields.push_back(f);
    } else if (c->pde == GBS_WAVE3D) {
        fields = {0};
    } else {
        fields = {0, 2};                        // acoustics: p and v cross the y slabs
    }
    const int nloc = c->loopback;
    const int S = c->slabs * nloc;              // global slab count
    if (c->slabs == 1) {
        // all slabs local: device-to-device copies
        for (int v = 0; v < nloc; ++v) {
            Slab& me = c->slab[v];
            Slab& lo = c->slab[(v - 1 + nloc) % nloc];
            Slab& hi = c->slab[(v + 1) % nloc];
            for (int f : fields) {
                double* mine = field_ptr(c, me, b, f);
                // bottom ghosts <- lower neighbour's top interior planes
                CU(c, cudaMemcpyAsync(mine - G * P, field_ptr(c, lo, b, f) + (lo.nz - G) * P,
                                      cnt * sizeof(double), cudaMemcpyDeviceToDevice, st));
                // top ghosts <- upper neighbour's bottom interior planes
                CU(c, cudaMemcpyAsync(mine + me.nz * P, field_ptr(c, hi, b, f),
                                      cnt * sizeof(double), cudaMemcpyDeviceToDevice, st));
            }
        }
        return GBS_OK;
    }
    if (nloc != 1) return fail(c, GBS_E_UNSUPPORTED, "loopback slabs with multi-GPU slabs");
    (void)S;
    (void)cnt;
    auto& A = nccl::api();
    Slab& me = c->slab[0];
    unsigned fm = 0;
    for (int f : fields) fm |= 1u << f;
    const std::vector<gbs_halo_op> ops = halo_schedule(c->slabs, c->my_slab, me.nz, (int)G, fm);
    NC(c, A.GroupStart());
    for (const auto& op : ops) {
        double* p = field_ptr(c, me, b, op.field) + op.plane0 * P;
        const size_t n = (size_t)(op.planes * P);
        if (op.kind == 0) NC(c, A.Send(p, n, nccl::ncclFloat64, op.peer, c->comm_slab, st));
        else NC(c, A.Recv(p, n, nccl::ncclFloat64, op.peer, c->comm_slab, st));
    }
    NC(c, A.GroupEnd());
    return GBS_OK;
}

// ---------------------------------------------------------------------------
// timing instrumentation (event pairs on the context stream)
// ---------------------------------------------------------------------------
static int timed_begin(gbs_ctx* c, int cls, cudaEvent_t* end_ev) {
    KernelTimer& T = c->timer;
    if (T.used + 2 > T.ev.size()) {
        for (int i = 0; i < 256; ++i) {
            cudaEvent_t e;
            CU(c, cudaEventCreate(&e));
            T.ev.push_back(e);
        }
        T.cls.resize(T.ev.size() / 2);
    }
    CU(c, cudaEventRecord(T.ev[T.used], c->stream));
    T.cls[T.used / 2] = cls;
    *end_ev = T.ev[T.used + 1];
    T.used += 2;
    return GBS_OK;
}

// Planes next to a slab face need the ghost planes; the rest do not.  With slabs the
// halo exchange runs on the context's comm stream while the interior planes are computed
// on the context stream, and the two face bands follow once the exchange is in (event
// fork / join, also inside the captured graph).  B = the face band thickness.
static int64_t face_band(const gbs_ctx* c, const Slab& s) {
    if (c->pde == GBS_ACOUSTIC2D && c->use_bulk && s.tma_ok) return gbs::tma::TY;   // whole 16-row bands
    return c->R;
}

static bool overlap_halo(gbs_ctx* c) {
    if (c->ghost == 0 || !c->use_overlap) return false;
    for (const auto& s : c->slab)
        if (s.nz < 3 * face_band(c, s)) return false;
    return true;
}

static int comm_fork(gbs_ctx* c) {
    if (!c->cstream) {
        CU(c, cudaStreamCreateWithFlags(&c->cstream, cudaStreamNonBlocking));
        CU(c, cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
        CU(c, cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
    }
    CU(c, cudaEventRecord(c->ev_fork, c->stream));
    CU(c, cudaStreamWaitEvent(c->cstream, c->ev_fork, 0));
    return GBS_OK;
}

static int comm_join(gbs_ctx* c) {
    CU(c, cudaEventRecord(c->ev_join, c->cstream));
    CU(c, cudaStreamWaitEvent(c->stream, c->ev_join, 0));
    return GBS_OK;
}

template <typename Launch>
static int run_overlapped(gbs_ctx* c, Launch&& launch, const std::vector<std::pair<int, unsigned>>& halos) {
    int rc;
    if (!overlap_halo(c)) {
        for (auto& h : halos)
            if ((rc = exchange_halo(c, h.first, h.second))) return rc;
        for (auto& s : c->slab)
            if ((rc = launch(s, (int64_t)0, s.nz))) return rc;
        return GBS_OK;
    }
    if ((rc = comm_fork(c))) return rc;
    for (auto& h : halos)
        if ((rc = exchange_halo(c, h.first, h.second, c->cstream))) return rc;
    for (auto& s : c->slab) {
        const int64_t B = face_band(c, s);
        if ((rc = launch(s, B, s.nz - B))) return rc;                  // interior: no ghosts read
    }
    if ((rc = comm_join(c))) return rc;
    for (auto& s : c->slab) {
        const int64_t B = face_band(c, s);
        if ((rc = launch(s, (int64_t)0, B))) return rc;
        if ((rc = launch(s, s.nz - B, s.nz))) return rc;
    }
    return GBS_OK;
}

static int step(gbs_ctx* c, int cls, const StepOperands& op) {
    int rc;
    cudaEvent_t end = nullptr;
    if (c->time_kernels && (rc = timed_begin(c, cls, &end))) return rc;
    rc = run_overlapped(c, [&](Slab& s, int64_t lo, int64_t hi) { return launch_step(c, s, op, lo, hi); },
                        {{op.S, 0u}});
    if (rc) return rc;
    if (end) CU(c, cudaEventRecord(end, c->stream));
    return GBS_OK;
}

static int pair_step(gbs_ctx* c, int cls, const PairOperands& op) {
    int rc;
    cudaEvent_t end = nullptr;
    if (c->time_kernels && (rc = timed_begin(c, cls, &end))) return rc;
    // the pair kernel reads S_u and U with stencils
    rc = run_overlapped(c, [&](Slab& s, int64_t lo, int64_t hi) { return launch_pair(c, s, op, lo, hi); },
                        {{op.Su.b, 1u << op.Su.f}, {op.U.b, 1u << op.U.f}});
    if (rc) return rc;
    if (end) CU(c, cudaEventRecord(end, c->stream));
    return GBS_OK;
}

static bool fused_path(const gbs_ctx* c) {
    if (!(c->use_fuse && c->use_bulk && c->nbuf == 6)) return false;
    for (const auto& s : c->slab)
        if (!s.tma_ok) return false;
    return true;
}

static int harvest_timer(gbs_ctx* c) {
    KernelTimer& T = c->timer;
    if (!T.used) return GBS_OK;
    CU(c, cudaStreamSynchronize(c->stream));
    for (size_t i = 0; i < T.used; i += 2) {
        float ms = 0.f;
        CU(c, cudaEventElapsedTime(&ms, T.ev[i], T.ev[i + 1]));
        int k = T.cls[i / 2];
        T.total_ms[k] += ms;
        T.launches[k] += 1;
    }
    T.used = 0;
    return GBS_OK;
}

// ---------------------------------------------------------------------------
// one macro step (enqueue only)
// ---------------------------------------------------------------------------
static int enqueue_macro(gbs_ctx* c, double H) {
    const int Y = c->yb, ACC = 1 - c->yb, B = 2, C = 3;
    const int64_t l0 = c->launches;
    int rc;
    bool first = true;
    const bool fused = fused_path(c);
    for (size_t q = 0; q < c->my_seq.size(); ++q) {
        const int k = c->my_seq[q];
        const int n = c->nk_all[k];
        const double h = H / (double)n;
        const bool last = (q + 1 == c->my_seq.size());
        if (fused) {
            // FE (which also forms u_2), then n/2 launches of two substeps:
            // (LF1, LF2), ..., (LF_{n-1}, final).  Field slots: y1 -> buffer 2; the
            // u-levels rotate through (2,0)/(3,0) and (4,0)/(5,0); v_{odd} stays in
            // (2,1) and v_{even} in (3,1), both updated in place (pointwise reads).
            StepOperands fe{Y, Y, 2, gbs::MODE_FE, h, 0.0, false};
            fe.xu = Slot{3, 0};
            fe.cf2 = 2.0 * h;
            if ((rc = step(c, 1, fe))) return rc;                                            // y1, u2
            Slot Pv{Y, 1}, Su{2, 0}, Sv{2, 1}, U{3, 0};
            for (int p = 0; p < n / 2; ++p) {
                if (p + 1 < n / 2) {
                    const int nb = Su.b == 2 ? 4 : 2;
                    PairOperands op{Pv, Su, Sv, U, Slot{3, 1}, Slot{nb, 0}, Sv, Slot{nb + 1, 0},
                                    gbs::MODE_LF, 2.0 * h, 2.0 * h, 0.0, false};
                    if ((rc = pair_step(c, 3, op))) return rc;
                    Pv = Slot{3, 1}; Su = Slot{nb, 0}; U = Slot{nb + 1, 0};
                } else {
                    PairOperands fin{Pv, Su, Sv, U, Slot{ACC, 0}, Slot{ACC, 0}, Slot{ACC, 1}, Slot{ACC, 0},
                                     first ? gbs::MODE_FIN0 : gbs::MODE_FINACC, 2.0 * h, h,
                                     0.5 * c->wk_all[k], last};
                    if ((rc = pair_step(c, 4, fin))) return rc;
                }
            }
            first = false;
            continue;
        }
        if ((rc = step(c, 1, {Y, Y, B, gbs::MODE_FE, h, 0.0, false}))) return rc;            // y1
        if ((rc = step(c, 0, {B, Y, C, gbs::MODE_LF, 2.0 * h, 0.0, false}))) return rc;      // y2
        int prev = B, cur = C;
        for (int i = 2; i <= n - 1; ++i) {                                                    // y3..yN
            if ((rc = step(c, 0, {cur, prev, prev, gbs::MODE_LF, 2.0 * h, 0.0, false}))) return rc;
            std::swap(prev, cur);
        }
        StepOperands fin{cur, prev, ACC, first ? gbs::MODE_FIN0 : gbs::MODE_FINACC, h,
                         0.5 * c->wk_all[k], last};
        if ((rc = step(c, 2, fin))) return rc;
        first = false;
    }
    if (c->groups > 1) {
        auto& A = nccl::api();
        Slab& s = c->slab[0];
        NC(c, A.GroupStart());
        for (int f = 0; f < c->F; ++f) {
            double* p = field_ptr(c, s, ACC, f);
            NC(c, A.AllReduce(p, p, (size_t)(s.nz * c->plane), nccl::ncclFloat64, nccl::ncclSum,
                              c->comm_group, c->stream));
        }
        NC(c, A.GroupEnd());
    }
    c->yb = ACC;
    c->launches_per_macro = c->launches - l0;
    return GBS_OK;
}

// ---------------------------------------------------------------------------
// small 1-D grids: the whole run in one cluster launch (K6)
// ---------------------------------------------------------------------------

static bool persistent_path(const gbs_ctx* c) {
    const int m = (int)c->my_seq.size();
    return c->use_persistent && c->pde == GBS_ADV1D && c->world == 1 && c->loopback == 1 && m >= 1 &&
           m <= 16 && c->n[0] <= kClusterMaxN;
}

static int launch_cluster_run(gbs_ctx* c, int64_t macro_steps, double H) {
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

// ---------------------------------------------------------------------------
// asynchronous slab IO: the copies run on their own streams and overlap the
// macro steps of the context stream; the state moves between the staging
// buffers and Y by device-to-device copies on the context stream, ordered by
// events (IN: h2d -> ready -> D2D into Y -> free; OUT: D2D from Y -> ready ->
// d2h -> free).
// ---------------------------------------------------------------------------
static int async_setup(gbs_ctx* c) {
    if (!c->in_buf.empty()) return GBS_OK;
    if (!c->h2d) {
        CU(c, cudaStreamCreateWithFlags(&c->h2d, cudaStreamNonBlocking));
        CU(c, cudaStreamCreateWithFlags(&c->d2h, cudaStreamNonBlocking));
        for (cudaEvent_t* e : {&c->ev_in_ready, &c->ev_in_free, &c->ev_out_ready, &c->ev_out_free})
            CU(c, cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    }
    for (auto& s : c->slab) {
        const size_t bytes = sizeof(double) * (size_t)c->F * (size_t)(s.nz * c->plane);
        double *in = nullptr, *out = nullptr;
        if (cudaMalloc(&in, bytes) != cudaSuccess || cudaMalloc(&out, bytes) != cudaSuccess) {
            if (in) cudaFree(in);
            return fail(c, GBS_E_NOMEM, "cudaMalloc of 2 x %zu bytes (async IO staging) failed", bytes);
        }
        c->in_buf.push_back(in);
        c->out_buf.push_back(out);
    }
    // nothing is in flight yet: both staging buffers start free
    CU(c, cudaEventRecord(c->ev_in_free, c->stream));
    CU(c, cudaEventRecord(c->ev_out_free, c->stream));
    return GBS_OK;
}

// drop the staging buffers (their sizes follow the slab layout); streams and events stay
static void async_release(gbs_ctx* c) {
    if (c->h2d) cudaStreamSynchronize(c->h2d);
    if (c->d2h) cudaStreamSynchronize(c->d2h);
    for (double* p : c->in_buf) cudaFree(p);
    for (double* p : c->out_buf) cudaFree(p);
    c->in_buf.clear();
    c->out_buf.clear();
    c->pending_in = false;
}

// a staged incoming state becomes Y (in context-stream order)
static int consume_in(gbs_ctx* c) {
    if (!c->pending_in) return GBS_OK;
    CU(c, cudaStreamWaitEvent(c->stream, c->ev_in_ready, 0));
    for (size_t v = 0; v < c->slab.size(); ++v) {
        Slab& s = c->slab[v];
        const int64_t n = s.nz * c->plane;
        for (int f = 0; f < c->F; ++f)
            CU(c, cudaMemcpyAsync(field_ptr(c, s, c->yb, f), c->in_buf[v] + (int64_t)f * n,
                                  sizeof(double) * (size_t)n, cudaMemcpyDeviceToDevice, c->stream));
    }
    CU(c, cudaEventRecord(c->ev_in_free, c->stream));
    c->pending_in = false;
    return GBS_OK;
}

static int check_flag(gbs_ctx* c) {
    int h = 0;
    CU(c, cudaMemcpyAsync(&h, c->d_flag, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    CU(c, cudaStreamSynchronize(c->stream));
    if (h) {
        CU(c, cudaMemsetAsync(c->d_flag, 0, sizeof(int), c->stream));
        return fail(c, GBS_E_NONFINITE, "non-finite state after a macro step (H beyond the stability limit?)");
    }
    return GBS_OK;
}

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
extern "C" {

const char* gbs_strerror(int code) {
    switch (code) {
        case GBS_OK: return "ok";
        case GBS_E_INVAL: return "invalid argument";
        case GBS_E_WEIGHTS: return "invalid extrapolation weights";
        case GBS_E_STATE: return "state not written";
        case GBS_E_NOMEM: return "out of memory";
        case GBS_E_CUDA: return "CUDA error";
        case GBS_E_NCCL: return "NCCL error";
        case GBS_E_NONFINITE: return "non-finite state";
        case GBS_E_UNSUPPORTED: return "unsupported";
        default: return "unknown error";
    }
}

const char* gbs_last_error(const gbs_ctx* c) { return c ? c->err.c_str() : g_err.c_str(); }

int gbs_nccl_unique_id(void* out128) {
    if (!out128) return fail(nullptr, GBS_E_INVAL, "out128 is NULL");
    auto& A = nccl::api();
    if (!A.ok) return fail(nullptr, GBS_E_NCCL, "libnccl.so.2 not found");
    nccl::uid_t id;
    int r = A.GetUniqueId(&id);
    if (r) return fail(nullptr, GBS_E_NCCL, "ncclGetUniqueId: %s", A.GetErrorString(r));
    memcpy(out128, &id, 128);
    return GBS_OK;
}

void gbs_destroy(gbs_ctx* c) {
    if (!c) return;
    if (c->stream) cudaStreamSynchronize(c->stream);
    if (c->h2d) { cudaStreamSynchronize(c->h2d); cudaStreamDestroy(c->h2d); }
    if (c->cstream) { cudaStreamSynchronize(c->cstream); cudaStreamDestroy(c->cstream); }
    if (c->ev_fork) cudaEventDestroy(c->ev_fork);
    if (c->ev_join) cudaEventDestroy(c->ev_join);
    if (c->d2h) { cudaStreamSynchronize(c->d2h); cudaStreamDestroy(c->d2h); }
    for (cudaEvent_t e : {c->ev_in_ready, c->ev_in_free, c->ev_out_ready, c->ev_out_free})
        if (e) cudaEventDestroy(e);
    for (double* p : c->in_buf) cudaFree(p);
    for (double* p : c->out_buf) cudaFree(p);
    c->in_buf.clear();
    c->out_buf.clear();
    for (auto& g : c->gexec) if (g) cudaGraphExecDestroy(g);
    free_state(c);
    if (c->d_flag) cudaFree(c->d_flag);
    if (c->d_gather) cudaFree(c->d_gather);
    if (c->d_nk) cudaFree(c->d_nk);
    if (c->d_wh) cudaFree(c->d_wh);
    if (c->d_alpha) cudaFree(c->d_alpha);
    for (auto e : c->timer.ev) cudaEventDestroy(e);
    auto& A = nccl::api();
    if (A.ok) {
        if (c->comm_group) A.CommDestroy(c->comm_group);
        if (c->comm_slab) A.CommDestroy(c->comm_slab);
        if (c->comm_world) A.CommDestroy(c->comm_world);
    }
    if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
    delete c;
}

static int build_ctx(gbs_ctx* c) { return alloc_state(c); }

// Validate the grid and the scheme (weights only when w_k != NULL) into c.
static int validate(gbs_ctx* c, const gbs_grid* g, int stencil_order, int m, const int32_t* n_k,
                    const double* w_k) {
    c->pde = g->pde;
    if (g->pde == GBS_ADV1D) { c->ndim = 1; c->F = 1; }
    else if (g->pde == GBS_ACOUSTIC2D) { c->ndim = 2; c->F = 3; }
    else if (g->pde == GBS_WAVE3D) { c->ndim = 3; c->F = 2; }
    else return fail(c, GBS_E_INVAL, "grid.pde=%d is not a known PDE", g->pde);
    if (g->ndim != c->ndim) return fail(c, GBS_E_INVAL, "grid.ndim=%d does not match the PDE", g->ndim);
    if (stencil_order == 0) {
        // spectral derivative: 1-D advection on an even grid, whole run in
        // the cluster kernel (N <= kClusterMaxN, m <= 16, one GPU)
        if (g->pde != GBS_ADV1D)
            return fail(c, GBS_E_INVAL, "stencil_order=0 (spectral) is defined for GBS_ADV1D only");
        if (g->n[0] < 4 || g->n[0] % 2 || g->n[0] > kSpectralMaxN)
            return fail(c, GBS_E_INVAL, "spectral grid n[0]=%lld must be even, 4..%d", (long long)g->n[0],
                        kSpectralMaxN);
        if (m > 16) return fail(c, GBS_E_INVAL, "spectral runs one sequence per CTA of a cluster: m=%d > 16", m);
    } else if (stencil_order != 4 && stencil_order != 8) {
        return fail(c, GBS_E_INVAL, "stencil_order=%d (must be 4 or 8, or 0 = spectral)", stencil_order);
    }
    c->order = stencil_order;
    c->R = stencil_order / 2;
    for (int d = 0; d < 3; ++d) {
        c->n[d] = g->n[d];
        c->len[d] = g->length[d] == 0.0 ? 1.0 : g->length[d];
        if (d < c->ndim) {
            if (g->n[d] < 2 * c->R + 1)
                return fail(c, GBS_E_INVAL, "grid.n[%d]=%lld < 2r+1=%d", d, (long long)g->n[d], 2 * c->R + 1);
            if (g->n[d] > (int64_t)1 << 30)
                return fail(c, GBS_E_INVAL, "grid.n[%d]=%lld too large", d, (long long)g->n[d]);
            if (!(c->len[d] > 0.0) || !std::isfinite(c->len[d]))
                return fail(c, GBS_E_INVAL, "grid.length[%d] must be positive", d);
        } else if (g->n[d] != 1) {
            return fail(c, GBS_E_INVAL, "grid.n[%d] must be 1 for a %d-D PDE", d, c->ndim);
        }
    }
    c->points = c->n[0] * c->n[1] * c->n[2];
    c->nslow = c->n[c->ndim - 1];
    c->plane = c->points / c->nslow;

    if (m < 1 || m > 32) return fail(c, GBS_E_INVAL, "m=%d (must be 1..32)", m);
    std::vector<std::pair<int, double>> seq;
    for (int i = 0; i < m; ++i) {
        if (n_k[i] < 2 || n_k[i] % 2) return fail(c, GBS_E_INVAL, "n_k[%d]=%d must be even and >= 2", i, n_k[i]);
        if (n_k[i] > 1 << 20) return fail(c, GBS_E_INVAL, "n_k[%d]=%d too large", i, n_k[i]);
        for (int j = 0; j < i; ++j)
            if (n_k[j] == n_k[i]) return fail(c, GBS_E_INVAL, "n_k[%d]=n_k[%d]=%d duplicate", j, i, n_k[i]);
        if (w_k && !std::isfinite(w_k[i])) return fail(c, GBS_E_WEIGHTS, "w_k[%d] is not finite", i);
        seq.push_back({n_k[i], w_k ? w_k[i] : 0.0});
    }
    std::sort(seq.begin(), seq.end());
    if (w_k) {
        double sw = 0.0, sa = 0.0;
        for (auto& p : seq) { sw += p.second; sa += std::fabs(p.second); }
        if (!(std::fabs(sw - 1.0) <= 1e-12 * sa))
            return fail(c, GBS_E_WEIGHTS, "sum of weights = %.17g (must be 1 within 1e-12 * sum|w|)", sw);
    }
    for (auto& p : seq) { c->nk_all.push_back(p.first); c->wk_all.push_back(p.second); }
    return GBS_OK;
}

// Plan g groups x s slabs for (rank, world) into c (no device work).
static int make_plan(gbs_ctx* c, int rank, int world, int groups) {
    if (world < 1 || rank < 0 || rank >= world) return fail(c, GBS_E_INVAL, "rank=%d world=%d", rank, world);
    if (groups < 0 || (groups > 0 && world % groups))
        return fail(c, GBS_E_INVAL, "groups=%d must divide world=%d", groups, world);
    c->rank = rank;
    c->world = world;
    plan(c, groups);
    if (c->groups * c->slabs != c->world)
        return fail(c, GBS_E_INVAL, "no valid plan: groups=%d does not fit world=%d (m=%d, slowest axis %lld)",
                    groups, world, (int)c->nk_all.size(), (long long)c->nslow);
    c->my_group = c->rank / c->slabs;
    c->my_slab = c->rank % c->slabs;
    c->my_seq = partition(c->nk_all, c->groups)[c->my_group];
    return GBS_OK;
}

int gbs_halo_schedule(int slabs, int my_slab, int64_t nz_local, int ghost, uint32_t field_mask, gbs_halo_op* ops,
                      int max_ops, int* n_ops) {
    if (!n_ops || (max_ops > 0 && !ops)) return fail(nullptr, GBS_E_INVAL, "n_ops or ops is NULL");
    if (slabs < 1 || my_slab < 0 || my_slab >= slabs || ghost < 0 || nz_local < ghost)
        return fail(nullptr, GBS_E_INVAL, "slabs=%d my_slab=%d nz_local=%lld ghost=%d", slabs, my_slab,
                    (long long)nz_local, ghost);
    const std::vector<gbs_halo_op> v = halo_schedule(slabs, my_slab, nz_local, ghost, field_mask);
    *n_ops = (int)v.size();
    for (int i = 0; i < (int)v.size() && i < max_ops; ++i) ops[i] = v[i];
    return (int)v.size() <= max_ops ? GBS_OK : fail(nullptr, GBS_E_INVAL, "max_ops=%d < %d", max_ops, (int)v.size());
}

int gbs_plan(const gbs_grid* g, int stencil_order, int m, const int32_t* n_k, int world, int rank, int groups,
             gbs_plan_info* out) {
    if (!g || !n_k || !out) return fail(nullptr, GBS_E_INVAL, "grid, n_k or out is NULL");
    gbs_ctx c;
    int rc = validate(&c, g, stencil_order, m, n_k, nullptr);
    if (!rc) rc = make_plan(&c, rank, world, groups);
    if (rc) { g_err = c.err; return rc; }
    memset(out, 0, sizeof(*out));
    out->groups = c.groups;
    out->slabs = c.slabs;
    out->my_group = c.my_group;
    out->my_slab = c.my_slab;
    out->my_sequences = (int)c.my_seq.size();
    for (size_t i = 0; i < c.my_seq.size(); ++i) {
        out->my_n_k[i] = c.nk_all[c.my_seq[i]];
        out->my_substeps += c.nk_all[c.my_seq[i]] + 1;
    }
    out->critical_substeps = crit_path(c.nk_all, c.groups);
    const int64_t nzl = c.nslow / c.slabs;
    out->slab_z0 = c.my_slab * nzl;
    out->slab_nz = nzl;
    return GBS_OK;
}

int gbs_create(const gbs_grid* g, int stencil_order, int m, const int32_t* n_k, const double* w_k,
               const gbs_dist* dist, void* cuda_stream, gbs_ctx** out) {
    if (!out) return fail(nullptr, GBS_E_INVAL, "out is NULL");
    *out = nullptr;
    if (!g || !n_k || !w_k) return fail(nullptr, GBS_E_INVAL, "grid, n_k or w_k is NULL");
    gbs_ctx* c = new (std::nothrow) gbs_ctx();
    if (!c) return fail(nullptr, GBS_E_NOMEM, "host allocation failed");
    auto bail = [&](int code) { g_err = c->err; gbs_destroy(c); return code; };
    int rc0 = validate(c, g, stencil_order, m, n_k, w_k);
    if (rc0) return bail(rc0);

    // ---- device / stream
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1)
        return bail(fail(c, GBS_E_CUDA, "no CUDA device available (this library has no CPU path)"));
    if (dist) c->device = dist->device;
    else cudaGetDevice(&c->device);
    if (c->device < 0 || c->device >= ndev)
        return bail(fail(c, GBS_E_INVAL, "device %d out of range (%d devices)", c->device, ndev));
    if (cudaSetDevice(c->device) != cudaSuccess)
        return bail(fail(c, GBS_E_CUDA, "cudaSetDevice(%d) failed", c->device));
    cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, c->device);
    if (c->sms < 1) c->sms = 148;
    if (cuda_stream) c->stream = (cudaStream_t)cuda_stream;
    else {
        if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess)
            return bail(fail(c, GBS_E_CUDA, "cudaStreamCreate failed"));
        c->own_stream = true;
    }

    // ---- plan + communicators
    if ((rc0 = make_plan(c, dist ? dist->rank : 0, dist ? dist->world : 1, dist ? dist->groups : 0)))
        return bail(rc0);
    if (c->world > 1) {
        auto& A = nccl::api();
        if (!A.ok) return bail(fail(c, GBS_E_NCCL, "libnccl.so.2 not found"));
        nccl::uid_t id;
        memcpy(&id, dist->nccl_id, 128);
        int r = A.CommInitRank(&c->comm_world, c->world, id, c->rank);
        if (r) return bail(fail(c, GBS_E_NCCL, "ncclCommInitRank: %s", A.GetErrorString(r)));
        if (c->slabs > 1) {
            r = A.CommSplit(c->comm_world, c->my_group, c->my_slab, &c->comm_slab, nullptr);
            if (r) return bail(fail(c, GBS_E_NCCL, "ncclCommSplit(slab): %s", A.GetErrorString(r)));
        }
        if (c->groups > 1) {
            r = A.CommSplit(c->comm_world, c->my_slab, c->my_group, &c->comm_group, nullptr);
            if (r) return bail(fail(c, GBS_E_NCCL, "ncclCommSplit(group): %s", A.GetErrorString(r)));
        }
        c->use_graph = false;   // NCCL calls stay outside graphs
    }
    int rc = build_ctx(c);
    if (rc) return bail(rc);
    if (cudaStreamSynchronize(c->stream) != cudaSuccess) return bail(fail(c, GBS_E_CUDA, "init sync failed"));
    *out = c;
    return GBS_OK;
}

int gbs_set_option(gbs_ctx* c, const char* key, int64_t value) {
    if (!c || !key) return fail(c, GBS_E_INVAL, "ctx or key is NULL");
    std::string k(key);
    auto drop_graphs = [&]() {
        for (auto& g : c->gexec) if (g) { cudaGraphExecDestroy(g); g = nullptr; }
        c->graph_H = -1.0;
    };
    if (k == "graph") { c->use_graph = value != 0 && c->world == 1; drop_graphs(); return GBS_OK; }
    if (k == "time_kernels") { c->time_kernels = value != 0; drop_graphs(); return GBS_OK; }
    if (k == "overlap") { c->use_overlap = value != 0; drop_graphs(); return GBS_OK; }
    if (k == "zchunk") { c->zchunk_opt = (int)std::max<int64_t>(0, value); drop_graphs(); return GBS_OK; }
    if (k == "bulk") { c->use_bulk = value != 0; drop_graphs(); return GBS_OK; }
    if (k == "fuse") { c->use_fuse = value != 0; drop_graphs(); return GBS_OK; }
    if (k == "persistent") { c->use_persistent = value != 0; return GBS_OK; }
    if (k == "loopback") {
        if (value < 1) return fail(c, GBS_E_INVAL, "loopback must be >= 1");
        if (c->world > 1) return fail(c, GBS_E_UNSUPPORTED, "loopback needs a single-GPU context");
        if (c->ndim == 1 && value > 1) return fail(c, GBS_E_UNSUPPORTED, "1-D grids are not slabbed");
        if (c->nslow % value || c->nslow / value < c->R)
            return fail(c, GBS_E_INVAL, "loopback=%lld must divide the slowest axis (%lld) into slabs >= r",
                        (long long)value, (long long)c->nslow);
        cudaStreamSynchronize(c->stream);
        drop_graphs();
        async_release(c);
        free_state(c);
        if (c->d_flag) { cudaFree(c->d_flag); c->d_flag = nullptr; }
        c->loopback = (int)value;
        c->have_state = false;
        return alloc_state(c);
    }
    return fail(c, GBS_E_INVAL, "unknown option '%s'", key);
}

int gbs_write_state(gbs_ctx* c, const double* src, int64_t count, int on_device) {
    if (!c || !src) return fail(c, GBS_E_INVAL, "ctx or src is NULL");
    if (count != c->F * c->points)
        return fail(c, GBS_E_INVAL, "count=%lld, expected F*points=%lld", (long long)count, (long long)(c->F * c->points));
    CU(c, cudaSetDevice(c->device));
    int rc0 = consume_in(c);
    if (rc0) return rc0;
    const cudaMemcpyKind kind = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    for (auto& s : c->slab)
        for (int f = 0; f < c->F; ++f)
            CU(c, cudaMemcpyAsync(field_ptr(c, s, c->yb, f), src + (int64_t)f * c->points + s.z0 * c->plane,
                                  sizeof(double) * (size_t)(s.nz * c->plane), kind, c->stream));
    c->have_state = true;
    return GBS_OK;
}

int gbs_advance(gbs_ctx* c, int64_t macro_steps, double H) {
    if (!c) return fail(c, GBS_E_INVAL, "ctx is NULL");
    if (!c->have_state) return fail(c, GBS_E_STATE, "gbs_advance before gbs_write_state");
    if (macro_steps < 0) return fail(c, GBS_E_INVAL, "macro_steps=%lld < 0", (long long)macro_steps);
    if (!(H > 0.0) || !std::isfinite(H)) return fail(c, GBS_E_INVAL, "H=%g must be positive and finite", H);
    CU(c, cudaSetDevice(c->device));
    int rc;
    if ((rc = consume_in(c))) return rc;
    if (macro_steps > 0 && persistent_path(c)) {
        if ((rc = launch_cluster_run(c, macro_steps, H))) return rc;
        c->macro_done += macro_steps;
        c->t += H * (double)macro_steps;
        return GBS_OK;
    }
    if (c->order == 0)
        return fail(c, GBS_E_UNSUPPORTED, "the spectral derivative runs only in the cluster kernel "
                                          "(one GPU, no loopback, option persistent=1)");
    const bool graph = c->use_graph && !c->time_kernels && macro_steps > 0;
    if (graph && c->graph_H != H) {
        for (auto& g : c->gexec) if (g) { cudaGraphExecDestroy(g); g = nullptr; }
        c->graph_H = H;
    }
    for (int64_t i = 0; i < macro_steps; ++i) {
        if (graph) {
            const int par = c->yb;
            if (!c->gexec[par]) {
                cudaGraph_t gr;
                CU(c, cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
                rc = enqueue_macro(c, H);
                cudaError_t e = cudaStreamEndCapture(c->stream, &gr);
                if (rc) { if (e == cudaSuccess) cudaGraphDestroy(gr); return rc; }
                if (e != cudaSuccess) return fail(c, GBS_E_CUDA, "graph capture: %s", cudaGetErrorString(e));
                e = cudaGraphInstantiate(&c->gexec[par], gr, 0);
                cudaGraphDestroy(gr);
                if (e != cudaSuccess) return fail(c, GBS_E_CUDA, "graph instantiate: %s", cudaGetErrorString(e));
                c->yb = par;          // capture does not execute: rewind the parity
                c->launches -= c->launches_per_macro;
            }
            CU(c, cudaGraphLaunch(c->gexec[par], c->stream));
            c->launches += c->launches_per_macro;
            c->yb = 1 - par;
        } else {
            if ((rc = enqueue_macro(c, H))) return rc;
        }
        c->macro_done++;
        c->t += H;
    }
    return GBS_OK;
}

int gbs_sync(gbs_ctx* c) {
    if (!c) return fail(c, GBS_E_INVAL, "ctx is NULL");
    CU(c, cudaSetDevice(c->device));
    int rc = consume_in(c);
    if (rc) return rc;
    CU(c, cudaStreamSynchronize(c->stream));
    if (c->h2d) CU(c, cudaStreamSynchronize(c->h2d));
    if (c->d2h) CU(c, cudaStreamSynchronize(c->d2h));
    return check_flag(c);
}

int gbs_read_state(gbs_ctx* c, double* dst, int64_t count, int on_device) {
    if (!c || !dst) return fail(c, GBS_E_INVAL, "ctx or dst is NULL");
    if (!c->have_state) return fail(c, GBS_E_STATE, "gbs_read_state before gbs_write_state");
    if (count != c->F * c->points)
        return fail(c, GBS_E_INVAL, "count=%lld, expected F*points=%lld", (long long)count, (long long)(c->F * c->points));
    CU(c, cudaSetDevice(c->device));
    int rc0 = consume_in(c);
    if (rc0) return rc0;
    const cudaMemcpyKind kind = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    if (c->slabs == 1) {
        for (auto& s : c->slab)
            for (int f = 0; f < c->F; ++f)
                CU(c, cudaMemcpyAsync(dst + (int64_t)f * c->points + s.z0 * c->plane, field_ptr(c, s, c->yb, f),
                                      sizeof(double) * (size_t)(s.nz * c->plane), kind, c->stream));
    } else {
        auto& A = nccl::api();
        Slab& s = c->slab[0];
        const size_t slab_cnt = (size_t)(s.nz * c->plane);
        if (!c->d_gather) CU(c, cudaMalloc(&c->d_gather, sizeof(double) * (size_t)c->points));
        for (int f = 0; f < c->F; ++f) {
            NC(c, A.AllGather(field_ptr(c, s, c->yb, f), c->d_gather, slab_cnt, nccl::ncclFloat64,
                              c->comm_slab, c->stream));
            CU(c, cudaMemcpyAsync(dst + (int64_t)f * c->points, c->d_gather, sizeof(double) * (size_t)c->points,
                                  kind, c->stream));
        }
    }
    int rc = gbs_sync(c);
    if (rc) return rc;
    return harvest_timer(c);
}

// this rank's planes [z_lo, z_lo + nz_rank) of the slowest axis (all its local slabs)
static void rank_planes(const gbs_ctx* c, int64_t* z_lo, int64_t* nz_rank) {
    *z_lo = c->slab[0].z0;
    *nz_rank = 0;
    for (const auto& s : c->slab) *nz_rank += s.nz;
}

int gbs_write_slab(gbs_ctx* c, const double* src, int64_t count, int on_device) {
    if (!c || !src) return fail(c, GBS_E_INVAL, "ctx or src is NULL");
    int64_t z_lo, nzr;
    rank_planes(c, &z_lo, &nzr);
    const int64_t per_field = nzr * c->plane;
    if (count != c->F * per_field)
        return fail(c, GBS_E_INVAL, "count=%lld, expected F*slab points=%lld", (long long)count,
                    (long long)(c->F * per_field));
    CU(c, cudaSetDevice(c->device));
    int rc0 = consume_in(c);
    if (rc0) return rc0;
    const cudaMemcpyKind kind = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    for (auto& s : c->slab)
        for (int f = 0; f < c->F; ++f)
            CU(c, cudaMemcpyAsync(field_ptr(c, s, c->yb, f), src + (int64_t)f * per_field + (s.z0 - z_lo) * c->plane,
                                  sizeof(double) * (size_t)(s.nz * c->plane), kind, c->stream));
    c->have_state = true;
    return GBS_OK;
}

int gbs_read_slab(gbs_ctx* c, double* dst, int64_t count, int on_device) {
    if (!c || !dst) return fail(c, GBS_E_INVAL, "ctx or dst is NULL");
    if (!c->have_state) return fail(c, GBS_E_STATE, "gbs_read_slab before gbs_write_state/slab");
    int64_t z_lo, nzr;
    rank_planes(c, &z_lo, &nzr);
    const int64_t per_field = nzr * c->plane;
    if (count != c->F * per_field)
        return fail(c, GBS_E_INVAL, "count=%lld, expected F*slab points=%lld", (long long)count,
                    (long long)(c->F * per_field));
    CU(c, cudaSetDevice(c->device));
    int rc0 = consume_in(c);
    if (rc0) return rc0;
    const cudaMemcpyKind kind = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    for (auto& s : c->slab)
        for (int f = 0; f < c->F; ++f)
            CU(c, cudaMemcpyAsync(dst + (int64_t)f * per_field + (s.z0 - z_lo) * c->plane, field_ptr(c, s, c->yb, f),
                                  sizeof(double) * (size_t)(s.nz * c->plane), kind, c->stream));
    int rc = gbs_sync(c);
    if (rc) return rc;
    return harvest_timer(c);
}

int gbs_write_slab_async(gbs_ctx* c, const double* src, int64_t count, int on_device) {
    if (!c || !src) return fail(c, GBS_E_INVAL, "ctx or src is NULL");
    int64_t z_lo, nzr;
    rank_planes(c, &z_lo, &nzr);
    const int64_t per_field = nzr * c->plane;
    if (count != c->F * per_field)
        return fail(c, GBS_E_INVAL, "count=%lld, expected F*slab points=%lld", (long long)count,
                    (long long)(c->F * per_field));
    CU(c, cudaSetDevice(c->device));
    int rc;
    if ((rc = async_setup(c))) return rc;
    if ((rc = consume_in(c))) return rc;            // an earlier staged state lands first
    CU(c, cudaStreamWaitEvent(c->h2d, c->ev_in_free, 0));
    const cudaMemcpyKind kind = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    for (size_t v = 0; v < c->slab.size(); ++v) {
        Slab& s = c->slab[v];
        const int64_t n = s.nz * c->plane;
        for (int f = 0; f < c->F; ++f)
            CU(c, cudaMemcpyAsync(c->in_buf[v] + (int64_t)f * n, src + (int64_t)f * per_field + (s.z0 - z_lo) * c->plane,
                                  sizeof(double) * (size_t)n, kind, c->h2d));
    }
    CU(c, cudaEventRecord(c->ev_in_ready, c->h2d));
    c->pending_in = true;
    c->have_state = true;
    return GBS_OK;
}

int gbs_read_slab_async(gbs_ctx* c, double* dst, int64_t count, int on_device) {
    if (!c || !dst) return fail(c, GBS_E_INVAL, "ctx or dst is NULL");
    if (!c->have_state) return fail(c, GBS_E_STATE, "gbs_read_slab_async before a state was written");
    int64_t z_lo, nzr;
    rank_planes(c, &z_lo, &nzr);
    const int64_t per_field = nzr * c->plane;
    if (count != c->F * per_field)
        return fail(c, GBS_E_INVAL, "count=%lld, expected F*slab points=%lld", (long long)count,
                    (long long)(c->F * per_field));
    CU(c, cudaSetDevice(c->device));
    int rc;
    if ((rc = async_setup(c))) return rc;
    if ((rc = consume_in(c))) return rc;
    // snapshot Y into the outgoing staging buffer (context stream), then copy it out (d2h)
    CU(c, cudaStreamWaitEvent(c->stream, c->ev_out_free, 0));
    for (size_t v = 0; v < c->slab.size(); ++v) {
        Slab& s = c->slab[v];
        const int64_t n = s.nz * c->plane;
        for (int f = 0; f < c->F; ++f)
            CU(c, cudaMemcpyAsync(c->out_buf[v] + (int64_t)f * n, field_ptr(c, s, c->yb, f),
                                  sizeof(double) * (size_t)n, cudaMemcpyDeviceToDevice, c->stream));
    }
    CU(c, cudaEventRecord(c->ev_out_ready, c->stream));
    CU(c, cudaStreamWaitEvent(c->d2h, c->ev_out_ready, 0));
    const cudaMemcpyKind kind = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    for (size_t v = 0; v < c->slab.size(); ++v) {
        Slab& s = c->slab[v];
        const int64_t n = s.nz * c->plane;
        for (int f = 0; f < c->F; ++f)
            CU(c, cudaMemcpyAsync(dst + (int64_t)f * per_field + (s.z0 - z_lo) * c->plane, c->out_buf[v] + (int64_t)f * n,
                                  sizeof(double) * (size_t)n, kind, c->d2h));
    }
    CU(c, cudaEventRecord(c->ev_out_free, c->d2h));
    return GBS_OK;
}

int gbs_query(const gbs_ctx* c, gbs_info* info) {
    if (!c || !info) return fail(const_cast<gbs_ctx*>(c), GBS_E_INVAL, "ctx or info is NULL");
    memset(info, 0, sizeof(*info));
    info->m = (int)c->nk_all.size();
    info->fields = c->F;
    info->radius = c->R;
    info->groups = c->groups;
    info->slabs = c->slabs * c->loopback;
    info->my_group = c->my_group;
    info->my_slab = c->my_slab;
    info->my_sequences = (int)c->my_seq.size();
    info->uses_graph = c->use_graph && !c->time_kernels;
    int64_t S = 0, mine = 0;
    for (int n : c->nk_all) S += n + 1;
    for (int k : c->my_seq) mine += c->nk_all[k] + 1;
    info->substeps_per_macro = S;
    info->my_substeps = mine;
    info->slab_z0 = c->slab.empty() ? 0 : c->slab[0].z0;
    info->slab_nz = c->slab.empty() ? 0 : c->slab[0].nz * c->loopback;
    info->points = c->points;
    info->macro_steps_done = c->macro_done;
    info->kernel_launches = c->launches;
    info->t = c->t;
    info->bytes_per_point_substep = 24.0 * c->F;
    return GBS_OK;
}

int gbs_kernel_time(gbs_ctx* c, int cls, double* total_ms, int64_t* launches, int reset) {
    if (!c || cls < 0 || cls > 5) return fail(c, GBS_E_INVAL, "ctx NULL or cls out of range");
    int rc = harvest_timer(c);
    if (rc) return rc;
    if (total_ms) *total_ms = c->timer.total_ms[cls];
    if (launches) *launches = c->timer.launches[cls];
    if (reset) { c->timer.total_ms[cls] = 0; c->timer.launches[cls] = 0; }
    return GBS_OK;
}

}  // extern "C"

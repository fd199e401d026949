// gbs_internal.h -- state and helpers shared by the translation units of
// libgbs_b200.so (not part of the C ABI; every symbol here has hidden
// visibility).  gbs_api.cu: context lifetime, options, queries; gbs_plan.cu:
// validation, the sequence-group x slab planner, the halo schedule;
// gbs_launch.cu: device memory, tensor maps and every kernel launch;
// gbs_exec.cu: the macro-step schedule (halo exchange, comm/compute overlap,
// CUDA graphs); gbs_io.cu: synchronous and asynchronous state IO.
#pragma once

#include "gbs.h"

#include <cuda.h>
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
Api& api();                        // gbs_api.cu
}  // namespace nccl

namespace cufft {
// cuFFT, resolved at run time (the process's libcufft.so.11, e.g. torch's) for the spectral
// derivative on grids beyond the cluster kernel; plans are made once per context
typedef int handle_t;
enum { D2Z = 0x6a, Z2D = 0x6c };
typedef int (*Plan1d_t)(handle_t*, int, int, int);
typedef int (*ExecD2Z_t)(handle_t, double*, void*);
typedef int (*ExecZ2D_t)(handle_t, void*, double*);
typedef int (*SetStream_t)(handle_t, cudaStream_t);
typedef int (*Destroy_t)(handle_t);
struct Api {
    bool ok = false;
    Plan1d_t Plan1d; ExecD2Z_t ExecD2Z; ExecZ2D_t ExecZ2D; SetStream_t SetStream; Destroy_t Destroy;
};
Api& api();                        // gbs_api.cu
}  // namespace cufft

// ---------------------------------------------------------------------------
// Collectives of the macro step (gbs_comm.cu): NCCL (one process per GPU) or the
// in-process local transport (every rank a context of this process on one device).
// ---------------------------------------------------------------------------
struct gbs_ctx;
struct Comm {
    int rank = 0, size = 1;
    virtual ~Comm() {}
    virtual bool is_nccl() const = 0;
    // grouped point-to-point (the halo planes): posted between group_start and group_end
    virtual int group_start(gbs_ctx* c) = 0;
    virtual int send(gbs_ctx* c, const double* p, size_t n, int peer, cudaStream_t st) = 0;
    virtual int recv(gbs_ctx* c, double* p, size_t n, int peer, cudaStream_t st) = 0;
    virtual int group_end(gbs_ctx* c, cudaStream_t st) = 0;
    // in place: p[i][0..n[i]) <- sum over the members (k buffers, one collective group)
    virtual int allreduce_sum(gbs_ctx* c, double* const* p, const size_t* n, int k, cudaStream_t st) = 0;
    // dst[j*n .. (j+1)*n) <- member j's src
    virtual int allgather(gbs_ctx* c, const double* src, double* dst, size_t n, cudaStream_t st) = 0;
    virtual int split(gbs_ctx* c, int color, int key, Comm** out) = 0;
    // device-side barrier of the members on stream st: work enqueued after it runs after every
    // member's work enqueued before it (local: events + host barrier; NCCL: a 1-value all-reduce)
    virtual int fence(gbs_ctx* c, cudaStream_t st) = 0;
    // member i's context when the members share this process (local transport), else nullptr
    virtual gbs_ctx* member_ctx(int) { return nullptr; }
    virtual void register_ctx(gbs_ctx*) {}
    // local transport: wake every member blocked in a collective of this communicator with an
    // error (a rank that failed will not arrive); NCCL: nothing (ncclCommAbort is the caller's)
    virtual void abort() {}
};
int comm_init(gbs_ctx* c, const gbs_dist* d);   // world, slab and group communicators
int comm_nccl_self(gbs_ctx* c, Comm** out);      // one-rank NCCL communicator (loopback_nccl)
void comm_release(gbs_ctx* c);
int comm_abort_on_error(gbs_ctx* c, int rc);     // rc != GBS_OK: abort the local communicators

// ---------------------------------------------------------------------------
struct Slab {
    int64_t z0 = 0, nz = 0;           // interior planes [z0, z0 + nz) of the slowest axis
    double* buf[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};   // Y, ACC, L0..L3 (+ ghosts)
    bool tma_ok = false;              // tensor maps below are valid (TMA kernels eligible)
    // [buffer][field][box]: 64x16, 64xr, rx16 (all TMA kernels); the 2-D chain kernels also
    // 64xBH, rxBH, 64x(BH+2r), rx(BH+2r), 64x(BH+4r), rx(BH+4r) (BH = tma::AC2_BH = 32 rows)
    CUtensorMap tm[6][3][9];
};

constexpr int kClusterMaxN = 7000;     // 4 nx doubles of shared memory per CTA
constexpr int kSpectralMaxN = 6400;    // 4.5 nx doubles (state, levels, weights)

struct KernelTimer {
    std::vector<cudaEvent_t> ev;      // pairs
    std::vector<int> cls;
    size_t used = 0;
    double total_ms[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    int64_t launches[8] = {0, 0, 0, 0, 0, 0, 0, 0};
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
    Comm* comm_world = nullptr;       // all ranks
    Comm* comm_slab = nullptr;        // the slabs of this rank's sequence group (halo exchange, gather)
    Comm* comm_group = nullptr;       // the groups holding this rank's slab (combine)
    bool local_transport = false;     // ranks are contexts of this process (gbs_local_hub_create)
    // fused combine across sequence groups (option "fused_combine"): the last
    // final pass of each group stores its w-scaled partial of owner j's plane range straight
    // into j's staging slot; each owner sums its range in member order and stores the sum into
    // every member's accumulator (reduce-scatter + all-gather without a collective call)
    bool fused_combine = false;
    double* d_stage = nullptr;        // [source group][field][planes of my range][plane]
    int64_t stage_doubles = 0;
    double* d_fence = nullptr;        // NCCL fence operand (Comm::fence)
    // gbs_bind_group_peers: every group member's workspace and staging buffer mapped into this
    // process (peer memory across GPUs); empty = the members' contexts (local transport)
    std::vector<char*> grp_ws, grp_stage;
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
    int fft_fwd = -1, fft_inv = -1;   // cuFFT D2Z / Z2D plans (order 0 beyond the cluster kernel)
    double* fft_buf = nullptr;        // N/2 + 1 complex spectrum, then the N-point derivative
    // asynchronous slab IO (gbs_write_slab_async / gbs_read_slab_async): per local slab a
    // staging buffer for the incoming and for the outgoing state, own copy streams
    std::vector<double*> in_buf, out_buf;
    cudaStream_t h2d = nullptr, d2h = nullptr;
    cudaEvent_t ev_in_ready = nullptr, ev_in_free = nullptr, ev_out_ready = nullptr, ev_out_free = nullptr;
    bool pending_in = false;
    // state buffers: carved from a caller-bound workspace (gbs_bind_workspace) or owned
    bool buffers_ready = false;
    void* ws_ptr = nullptr;
    int64_t ws_bytes = 0;
    // halo exchange overlapped with the interior planes (slabbed layouts)
    bool use_overlap = true;
    cudaStream_t cstream = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    int* d_nk = nullptr;              // step counts / half weights for the cluster kernel
    double* d_wh = nullptr;
    bool use_fuse = true;             // two-substep (temporally blocked) kernels where eligible
    bool use_fuse2d = false;          // 2-D chain pair kernels (measured slower: opt-in)
                                      // (bit-exact)
    bool tma_grid = false;            // grid is a multiple of the TMA tile (wave3d)
    int nbuf = 4;                     // state buffers per slab: Y, ACC + 2 or 4 level buffers
    int zchunk_opt = 0;
    int zchunk_pair_opt = 0;          // planes per CTA of the two-substep kernel (0 = zchunk, else 256)
    int zchunk_fin_opt = 0;           // the same for its LF + final pass only (0 = as above)
    int hint_fin_opt = 11;            // L2 policy bits of the LF + final pass (PairArgs::hint)
    int n_streams = 1;                // sequence streams (option "streams": 1 or 2)
    bool fea_ring = true;             // that pass with both fields fed through tile rings (C5: 10.8
                                      // vs 11.0-11.3 ms per launch)
    bool fin_ring = false;            // the LF + final pass fed through tile rings (only 2 stages
                                      // fit: 13.1 vs 12.95 ms, off)
    bool use_fea = true;              // FE fused with chain A's first step (option "fea"; C5:
                                      // 12.3 ms instead of 7.55 + 5.96, macro step 506 -> 492 ms)
    cudaStream_t stream2 = nullptr;
    cudaEvent_t ev_fork2 = nullptr, ev_join2 = nullptr, ev_fin = nullptr;
    int hint_opt = 11;                // pair kernel L2 policy bits (PairArgs::hint)
    int hint_step_opt = 0;            // single-step 3-D TMA kernel L2 policy bits (Wave3DArgs::hint)
    bool use_half = true;             // leap-frog pairs as two single-stencil-field launches, FE
                                      // through the same kernel (gbs_wave3d_half.cuh)
    bool half_tall = true;            // 64 x 32 tiles when ny allows
    int half_rpt = 4;                 // rows per thread of the tall half kernel (2 or 4; 4 measured
                                      // 2% faster on C5: 5.96 vs 6.10 ms per half)
    bool half_fe = false;             // FE through the half kernel (7.7 ms vs 7.5 for the FE step
                                      // kernel on C5: off by default)
    int hint_half_opt = 11;           // half kernel L2 / streaming bits (HalfArgs::hint)
    bool loop_nccl = false;           // loopback halos through NCCL on a one-rank communicator
    // peer halo pushes (gbs_wave3d_tma.cuh PeerPush): option "peer" (loopback slabs) or
    // gbs_bind_peers (one slab per GPU, neighbours' workspaces mapped into this process)
    bool peer_on = false;
    bool peer_ghosts_valid = false;   // Y's ghost planes hold the neighbours' current face planes
    unsigned long long peer_epoch = 0;
    bool peer_flags_fresh = false;    // this rank's flags were zeroed by gbs_bind_workspace
    char* peer_base[2] = {nullptr, nullptr};   // lower / upper neighbour's workspace (multi-GPU)
    unsigned long long* d_peer_flags = nullptr; // loopback: [slab][from lower, from upper]
    int band_opt = 0;                 // 3-D TMA tile launch order (0 = whole rows)
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

extern thread_local std::string g_err;
int fail(gbs_ctx* c, int code, const char* fmt, ...);

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
// memory helpers
// ---------------------------------------------------------------------------
inline double* field_ptr(gbs_ctx* c, Slab& s, int b, int f) {
    return s.buf[b] + (int64_t)f * c->field_stride + c->ghost * c->plane;
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
    // FIN modes: store the result here instead of the accumulator buffer (plane z at
    // out_u + z * plane; the accumulator is still read from Bu.b) -- the fused combine
    double* out_u = nullptr;
    double* out_v = nullptr;
};

// One single-stencil-field 3-D launch (gbs_wave3d_half.cuh): O1 = P + c1 lap(X),
// O2 = X + c2 O1 (+ O3 = X + c1 P for the forward-Euler kind).
struct HalfOperands {
    int kind;             // gbs::tma::HALF_LF or HALF_FE
    Slot X, P, O1, O2;
    Slot O3 = {-1, 0};
    double c1 = 0.0, c2 = 0.0;
};

// ---- gbs_plan.cu
std::vector<std::vector<int>> partition(const std::vector<int>& nk, int g);
int64_t crit_path(const std::vector<int>& nk, int g);
void plan(gbs_ctx* c, int want_groups);
std::vector<gbs_halo_op> halo_schedule(int slabs, int my_slab, int64_t nz, int G, unsigned mask);
int validate(gbs_ctx* c, const gbs_grid* g, int stencil_order, int m, const int32_t* n_k, const double* w_k);
int make_plan(gbs_ctx* c, int rank, int world, int groups);
// ---- gbs_launch.cu
int alloc_state(gbs_ctx* c);            // layout + flag; buffers on first use
int ensure_buffers(gbs_ctx* c);         // allocate (or carve) the state buffers, tensor maps
int64_t state_bytes(const gbs_ctx* c);  // device bytes of the state buffers of this layout
void free_state(gbs_ctx* c);
// [lo, hi) of slab s; gap > 0: only the two face bands of (hi - lo - gap) / 2 planes each
int launch_step(gbs_ctx* c, Slab& s, const StepOperands& op, int64_t lo, int64_t hi, int64_t gap = 0);
int launch_pair(gbs_ctx* c, Slab& s, const PairOperands& op, int64_t lo, int64_t hi, int64_t gap = 0);
int launch_half(gbs_ctx* c, Slab& s, const HalfOperands& op, int64_t lo, int64_t hi, int64_t gap = 0);
bool half_eligible(const gbs_ctx* c);
// ghost rows of a single slab from its own opposite side, for (buffer, field mask) pairs
int launch_ghost_fill(gbs_ctx* c, const std::vector<std::pair<int, unsigned>>& halos);
// 2-D acoustics, two leap-frog substeps (P, S buffers -> A = y_{n+1}, B = y_{n+2} buffers)
int launch_ac2d_pair(gbs_ctx* c, Slab& s, int P, int S, int Aout, int Bout, double cfA, double cfB, int64_t lo,
                     int64_t hi, int64_t gap = 0);
bool persistent_path(const gbs_ctx* c);
double* peer_field(gbs_ctx* c, int v, int side, int b, int f);   // neighbour's field base
unsigned long long* peer_flag(gbs_ctx* c, int v, int which);       // this slab's flag (0 lo, 1 hi)
unsigned long long* peer_flag_remote(gbs_ctx* c, int v, int side); // the flag a neighbour waits on
int peer_eligible(const gbs_ctx* c, bool multi_gpu);
constexpr int64_t kPeerFlagBytes = 256;    // workspace tail: this rank's two flags (multi-GPU)
int spectral_setup(gbs_ctx* c);       // cuFFT plans + buffers (order 0); idempotent
void spectral_release(gbs_ctx* c);
int launch_cluster_run(gbs_ctx* c, int64_t macro_steps, double H);
// ---- gbs_comm.cu
int owner_combine(gbs_ctx* c, double* const* in, double* const* out, int n, int64_t count, cudaStream_t st);
// ---- gbs_exec.cu
int64_t stage_bytes_of(const gbs_ctx* c);     // staging buffer of the fused combine
int timed_begin(gbs_ctx* c, int cls, cudaEvent_t* end_ev);
int harvest_timer(gbs_ctx* c);
// ---- gbs_io.cu
void async_release(gbs_ctx* c);
int consume_in(gbs_ctx* c);
int check_flag(gbs_ctx* c);

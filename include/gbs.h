/*
 * gbs.h -- C ABI of the B200-native extrapolated GBS hot path
 *          (libgbs_b200.so, built from paper_1907_11771_b200/csrc).
 *
 * What it computes (§2.1, Eq. (1) "eq:GBS", lines 85-98, and the
 * Richardson combination, lines 109-115 and 221-225; App. B R = sum c_i P_i,
 * line 679): for every macro step ("section") of length H, starting from the
 * current state Y, each of the m sequences k runs
 *
 *     y_1     = y_0 + h f(y_0),            h = H / n_k, y_0 = Y       (FE)
 *     y_{n+1} = y_{n-1} + 2h f(y_n),       n = 1..n_k                 (LF)
 *     y*_k    = (y_{n_k-1} + 2 y_{n_k} + y_{n_k+1}) / 4               (averaging)
 *
 * and the new state is  Y <- sum_k w_k y*_k,  summed in ascending n_k order.
 * f is the method-of-lines right-hand side of a built-in linear PDE on a
 * periodic box with centered finite differences of order 4 or 8
 * (BASELINE.json configs) or, for GBS_ADV1D, the paper's own spectral
 * (Fourier collocation) derivative (stencil_order 0; §4.1):
 *
 *     GBS_ADV1D       u_t = -u_x                                   F = 1
 *     GBS_ACOUSTIC2D  p_t = -(u_x + v_y), u_t = -p_x, v_t = -p_y    F = 3
 *     GBS_WAVE3D      u_t = v, v_t = u_xx + u_yy + u_zz             F = 2
 *
 * All arithmetic is IEEE fp64.  Every step above runs on the GPU, in this
 * library's CUDA kernels (sm_100a) -- with one exception: the spectral
 * derivative on grids beyond the cluster kernel (n[0] > 6400, or m > 16, or
 * sequence groups across GPUs) transforms with cuFFT (D2Z / Z2D, a library
 * call; the i k scaling and every substep update are this library's kernels).
 * There is no CPU fallback: without a usable CUDA device gbs_create fails with
 * GBS_E_CUDA.
 *
 * State layout (host or device, caller-owned): SoA fp64, [F][nz][ny][nx],
 * x fastest, unused axes of extent 1; count = F * nx * ny * nz values.
 * Grid point i of axis d sits at i * length[d] / n[d] (periodic, S6).
 *
 * Ownership: the context owns every device buffer it allocates; caller
 * arrays are read or written only during the call (never retained).  A
 * context is not thread-safe; distinct contexts are independent.  No C++
 * exception crosses this ABI; every int-returning call returns GBS_OK (0) or
 * a negative GBS_E_* code, and gbs_last_error(ctx) explains the last failure.
 */
#ifndef GBS_B200_H
#define GBS_B200_H

#include <stdint.h>

#if defined(__GNUC__)
#define GBS_API __attribute__((visibility("default")))
#else
#define GBS_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ------------------------------------------------------ */
#define GBS_OK            0
#define GBS_E_INVAL      -1   /* bad argument: odd/duplicate/<2 n_k, m outside [1,32],
                                 stencil order not 4/8, n[d] < 2r+1, H <= 0 or non-finite,
                                 count mismatch, NULL pointer (named in gbs_last_error) */
#define GBS_E_WEIGHTS    -2   /* non-finite weight, or |sum w - 1| > 1e-12 * sum |w|
                                 (first row of Eq. (3)) */
#define GBS_E_STATE      -3   /* gbs_advance / gbs_read_state before gbs_write_state */
#define GBS_E_NOMEM      -4   /* device (or pinned host) allocation failed */
#define GBS_E_CUDA       -5   /* CUDA runtime error, or no CUDA device */
#define GBS_E_NCCL       -6   /* NCCL error (multi-GPU contexts) */
#define GBS_E_NONFINITE  -7   /* a macro step produced a non-finite value (instability:
                                 H beyond the imaginary stability boundary); reported by
                                 the gbs_sync / gbs_read_state after it happened */
#define GBS_E_UNSUPPORTED -8  /* valid request this build does not implement */

/* ---- problem description ----------------------------------------------- */
#define GBS_ADV1D       1
#define GBS_ACOUSTIC2D  2
#define GBS_WAVE3D      3

typedef struct gbs_grid {
    int32_t pde;        /* GBS_ADV1D | GBS_ACOUSTIC2D | GBS_WAVE3D */
    int32_t ndim;       /* must equal the PDE's dimension (1, 2, 3) */
    int64_t n[3];       /* grid points (nx, ny, nz); unused axes = 1 */
    double  length[3];  /* periodic box side per axis; 0 means 1.0 (unit box) */
} gbs_grid;

/* Multi-GPU description (one process per GPU).  Pass NULL for a single GPU. */
#define GBS_TRANSPORT_NCCL   0   /* one process per GPU, NCCL communicators (production) */
#define GBS_TRANSPORT_LOCAL  1   /* every rank is a context of this process on ONE device,
                                    driven by its own host thread; collectives are device
                                    copies ordered by events and host barriers (tests and
                                    emulation of N ranks on one GPU; gbs_local_hub_create) */
typedef struct gbs_dist {
    int32_t rank;            /* this process's rank in [0, world) */
    int32_t world;           /* number of GPUs / processes */
    int32_t device;          /* CUDA device ordinal this rank uses */
    int32_t groups;          /* sequence groups g (world % g == 0); 0 = planner's choice.
                                world / g ranks share each group as z-slabs (y in 2-D) */
    uint8_t nccl_id[128];    /* ncclUniqueId made by gbs_nccl_unique_id on rank 0 and
                                broadcast by the caller (e.g. torch.distributed) */
    int32_t transport;       /* GBS_TRANSPORT_NCCL (0) or GBS_TRANSPORT_LOCAL */
    int32_t pad;
    void*   hub;             /* GBS_TRANSPORT_LOCAL: the hub shared by the world's contexts */
} gbs_dist;

/* In-process transport for `world` contexts on one device (GBS_TRANSPORT_LOCAL): create the
 * hub once, pass it in every rank's gbs_dist, call gbs_create / gbs_advance / gbs_read_state
 * of the ranks from `world` concurrent host threads (collectives block until every member of
 * the communicator arrives; a member whose gbs_advance / gbs_read_state fails releases them at
 * once, and one missing for 300 s fails them, both with GBS_E_NCCL), destroy
 * the hub after every context.  The macro step runs the same plan, halo schedule, group
 * combine and gather as over NCCL: halo planes by device-to-device copies matched in NCCL's
 * posting order, the combine as one kernel per rank that sums its share of the elements over
 * the group members in member order and stores the sum into every member (deterministic).
 * No kernel waits on another rank's kernel.  Not a performance path: the ranks share one GPU. */
GBS_API int gbs_local_hub_create(int world, int device, void** hub);
GBS_API void gbs_local_hub_destroy(void* hub);

/* Plan and accounting, filled by gbs_query. */
typedef struct gbs_info {
    int32_t m;                   /* number of sequences */
    int32_t fields;              /* F */
    int32_t radius;              /* stencil radius r */
    int32_t groups, slabs;       /* plan: g sequence groups x s slabs, g * s = world */
    int32_t my_group, my_slab;
    int32_t my_sequences;        /* sequences run by this rank */
    int32_t uses_graph;          /* 1 if the macro step is replayed as a CUDA graph */
    int64_t substeps_per_macro;  /* S = sum_k (n_k + 1): RHS-evaluating substeps */
    int64_t my_substeps;         /* substeps this rank runs per macro step (its group's) */
    int64_t slab_z0, slab_nz;    /* this rank's slab along the slowest axis */
    int64_t points;              /* nx * ny * nz (global) */
    int64_t macro_steps_done;
    int64_t kernel_launches;     /* kernels launched by this context so far */
    double  t;                   /* sum of H over completed gbs_advance calls */
    double  bytes_per_point_substep;  /* algorithmic HBM bytes: 24 F */
} gbs_info;

typedef struct gbs_ctx gbs_ctx;

/* A rank's share of the multi-GPU plan (gbs_plan; same planner as gbs_create). */
typedef struct gbs_plan_info {
    int32_t groups, slabs;         /* g sequence groups x s slabs, g * s = world */
    int32_t my_group, my_slab;     /* rank = my_group * slabs + my_slab */
    int32_t my_sequences;          /* sequences of this rank's group */
    int32_t my_n_k[32];            /* their step counts, ascending */
    int64_t my_substeps;           /* sum (n_k + 1) over them */
    int64_t critical_substeps;     /* max over groups of sum (n_k + 1) */
    int64_t slab_z0, slab_nz;      /* this rank's planes of the slowest axis */
} gbs_plan_info;

/* Host-only planning (no device, no NCCL): the sequence-group x slab plan that
 * gbs_create would use for (world, rank, groups) -- PAPER.md §3.6 (lines
 * 388-400) balances sequences by RHS evaluations; groups are balanced by
 * sum (n_k + 1) and the slowest axis is split into equal slabs.  Arguments as
 * gbs_create (weights are not needed); groups = 0 lets the planner choose. */
GBS_API int gbs_plan(const gbs_grid* grid, int stencil_order, int m, const int32_t* n_k, int world, int rank,
                     int groups, gbs_plan_info* out);

/* One point-to-point operation of the per-substep slab halo exchange. */
typedef struct gbs_halo_op {
    int32_t kind;       /* 0 = send, 1 = receive */
    int32_t peer;       /* slab index of the partner (rank in the slab communicator) */
    int32_t field;      /* state field (0 = u / p, 1 = v / u, 2 = v) */
    int32_t pad;
    int64_t plane0;     /* first local plane: interior planes are 0 .. nz_local-1, ghosts
                           are -ghost .. -1 (low side) and nz_local .. nz_local+ghost-1 */
    int64_t planes;     /* number of consecutive planes */
} gbs_halo_op;

/* Host-only: the ordered list of point-to-point operations one slab posts (inside
 * one ncclGroupStart/End) to refresh the ghost planes of the fields in field_mask
 * (bit f = field f) -- exactly the schedule gbs_advance uses.  For every pair of
 * slabs the k-th send from a to b lands in the k-th receive at b from a (NCCL
 * matches point-to-point operations in posting order), including slabs == 2,
 * where both neighbours are the same peer.  Writes at most max_ops entries to
 * ops and the number of operations to *n_ops. */
GBS_API int gbs_halo_schedule(int slabs, int my_slab, int64_t nz_local, int ghost, uint32_t field_mask,
                              gbs_halo_op* ops, int max_ops, int* n_ops);

/* Create a context: validate, plan, allocate, and (multi-GPU) join NCCL.
 *   grid           problem description (copied)
 *   stencil_order  4 or 8 (centered FD, radius r = order / 2), or 0: spectral
 *                  derivative of the trigonometric interpolant (GBS_ADV1D only,
 *                  n[0] even, >= 4).  n[0] <= 6400 with m <= 16 on one
 *                  GPU: one thread-block-cluster launch per gbs_advance (option
 *                  "persistent"); otherwise per substep cuFFT D2Z, i k scaling, Z2D
 *                  and the pointwise update (libcufft.so.11 resolved at run time;
 *                  GBS_E_UNSUPPORTED if absent)
 *   m, n_k, w_k    step counts (even, >= 2, distinct; 1 <= m <= 32) and their
 *                  fp64 weights (already rounded once from exact rationals by
 *                  the caller); both copied.  Sequences with
 *                  w_k == 0 are still executed (reading R3).
 *   dist           NULL, or the multi-GPU description above
 *   cuda_stream    cudaStream_t the context issues all work on (NULL = a
 *                  stream the context creates)
 *   out            receives the new context (NULL on failure)  */
GBS_API int gbs_create(const gbs_grid* grid, int stencil_order, int m, const int32_t* n_k,
               const double* w_k, const gbs_dist* dist, void* cuda_stream, gbs_ctx** out);

/* Load the state Y from src (count = F*nx*ny*nz values, full grid, SoA).
 * on_device = 1: src is device memory; 0: host memory (pinned or pageable).
 * Multi-GPU: every rank passes the full grid and keeps its own slab. */
GBS_API int gbs_write_state(gbs_ctx* ctx, const double* src, int64_t count, int on_device);

/* Advance Y by macro_steps (>= 0) macro steps of length H (> 0, finite).
 * Asynchronous on the context stream; t += macro_steps * H. */
GBS_API int gbs_advance(gbs_ctx* ctx, int64_t macro_steps, double H);

/* Copy the current Y (full grid) to dst; synchronizes the context stream and
 * surfaces deferred errors (GBS_E_NONFINITE).  Multi-GPU: every rank receives
 * the full grid (slabs are all-gathered). */
GBS_API int gbs_read_state(gbs_ctx* ctx, double* dst, int64_t count, int on_device);

/* Slab-local IO for multi-GPU callers that hold only their own part of the grid:
 * src/dst hold this rank's planes [slab_z0, slab_z0 + slab_nz) of the slowest axis
 * (gbs_query / gbs_plan) for every field, SoA [F][slab_nz][...], count = F * slab_nz *
 * plane.  Single GPU: the slab is the whole grid (identical to the full-grid calls).
 * gbs_read_slab synchronizes and surfaces deferred errors like gbs_read_state. */
GBS_API int gbs_write_slab(gbs_ctx* ctx, const double* src, int64_t count, int on_device);
GBS_API int gbs_read_slab(gbs_ctx* ctx, double* dst, int64_t count, int on_device);

/* Device memory.  The state buffers (F x points x 8 bytes each, 4 or 6 of them per local
 * slab incl. ghost planes) are allocated on the first write, by the context (cudaMalloc), or
 * carved out of a caller-owned workspace bound before that -- e.g. a torch tensor, so that
 * PyTorch's allocator owns the memory:
 *   gbs_workspace_bytes  bytes the current layout needs (depends on options such as loopback)
 *   gbs_bind_workspace   device_ptr (256-byte aligned, >= gbs_workspace_bytes) replaces the
 *                        context's own buffers (released); NULL returns to own buffers.  The
 *                        state is discarded: write it again.  The caller keeps the memory
 *                        alive and untouched until gbs_destroy or the next bind. */
GBS_API int gbs_workspace_bytes(const gbs_ctx* ctx, int64_t* bytes);
GBS_API int gbs_bind_workspace(gbs_ctx* ctx, void* device_ptr, int64_t bytes);

/* Peer halo pushes (pure z-slabs of the 3-D wave on a grid of whole
 * 64 x 16 tiles, two-substep path, one slab per GPU, groups = 1).  Instead of an NCCL halo
 * exchange before every substep, the kernel that produces a u-level stores its r face planes
 * straight into the neighbouring GPUs' ghost planes over NVLink, and a per-launch epoch flag
 * (release/acquire, system scope) orders each launch's face tiles after the neighbours'
 * previous launch (gbs_wave3d_tma.cuh, PeerPush).
 *   gbs_bind_peers  lower_workspace / upper_workspace: the workspaces (gbs_bind_workspace) of
 *                   the slab below / above, mapped into this process (e.g. torch symmetric
 *                   memory or CUDA IPC); every rank binds a workspace of the same layout, whose
 *                   last 256 bytes (part of gbs_workspace_bytes) hold the flags.  NULL, NULL returns to NCCL halos.
 *                   Graphs are not used while bound.  GBS_E_STATE without a workspace,
 *                   GBS_E_UNSUPPORTED when the layout does not qualify.
 * Option "peer" runs the same kernels and protocol between loopback slabs on one GPU.
 * Not yet run on more than one GPU. */
GBS_API int gbs_bind_peers(gbs_ctx* ctx, void* lower_workspace, void* upper_workspace);

/* Fused combine across sequence groups (the groups'
 * w-scaled partial sums are added).  The slab's planes are split into g owner ranges (range j =
 * planes [nz j / g, nz (j+1) / g) owned by group j).  The final pass of each group's last
 * sequence (3-D two-substep path) stores its partial sum of range j straight into owner j's
 * staging buffer (peer memory), each owner sums the g slots of its range in member order and
 * stores the sum into every member's accumulator -- a reduce-scatter and an all-gather with no
 * collective call; a device-side fence between the phases (local transport: events and host
 * barriers; NCCL: a one-value all-reduce on the group communicator).  Bit-identical to the
 * local transport's all-reduce (same sums in the same order).
 *   option "fused_combine" 1   the local transport (members are contexts of this process)
 *   gbs_stage_bytes            bytes of one member's staging buffer (g F max-range planes)
 *   gbs_bind_group_peers       member_workspaces[j] / member_stages[j]: group member j's bound
 *                              workspace (gbs_bind_workspace; same layout on every member) and
 *                              staging buffer, mapped into this process (e.g. torch symmetric
 *                              memory); member_workspaces[my_group] must be this context's own.
 *                              Turns the fused combine on; n = 0 turns it off.  GBS_E_STATE
 *                              without a workspace.  Not yet run across GPUs. */
GBS_API int gbs_stage_bytes(const gbs_ctx* ctx, int64_t* bytes);
GBS_API int gbs_bind_group_peers(gbs_ctx* ctx, void* const* member_workspaces, void* const* member_stages, int n);

/* Asynchronous slab IO (same layout and count as gbs_write_slab / gbs_read_slab; on one
 * GPU the slab is the whole grid).  The copies run on the context's own copy streams and
 * overlap the macro steps queued on the context stream:
 *   gbs_write_slab_async  stages src (pinned host or device) into a staging buffer; the
 *                         staged state becomes Y before the next gbs_advance / read / sync.
 *                         src must stay valid and unmodified until the next gbs_sync.
 *   gbs_read_slab_async   snapshots the current Y (after every macro step queued so far)
 *                         and copies it to dst; dst is complete after the next gbs_sync,
 *                         which also surfaces deferred errors.
 * Staging costs 2 x F x slab points x 8 bytes of device memory, allocated on first use.
 * A write-advance-read loop with these calls keeps the host<->device copies of one step
 * under the macro steps of the neighbouring ones. */
GBS_API int gbs_write_slab_async(gbs_ctx* ctx, const double* src, int64_t count, int on_device);
GBS_API int gbs_read_slab_async(gbs_ctx* ctx, double* dst, int64_t count, int on_device);

/* Wait for all queued work (compute and asynchronous copies); surfaces deferred errors. */
GBS_API int gbs_sync(gbs_ctx* ctx);

/* Release everything the context owns (NULL is a no-op). */
GBS_API void gbs_destroy(gbs_ctx* ctx);

/* Fill out128 with a fresh ncclUniqueId (call on rank 0, then broadcast). */
GBS_API int gbs_nccl_unique_id(void* out128);

/* Plan / accounting snapshot. */
GBS_API int gbs_query(const gbs_ctx* ctx, gbs_info* info);

/* Tuning and instrumentation knobs (key -> value); unknown keys -> GBS_E_INVAL.
 *   "graph"        1/0   replay each macro step as a CUDA graph (default 1)
 *   "time_kernels" 1/0   record a CUDA event pair around every stencil launch
 *                        (on the context stream) for gbs_kernel_time (default 0)
 *   "loopback"     s     emulate s z-slabs on this GPU with device-to-device
 *                        halo copies through the multi-GPU code path (tests)
 *   "bulk"         1/0   TMA-pipelined 3-D kernels on grids that are multiples of
 *                        their 64 x 16 tile (default 1; 0 = register-prefetch kernels)
 *   "fuse"         1/0   two substeps per HBM pass on 3-D TMA grids (default 1)
 *   "half"         1/0   3-D TMA grids: each two-substep leap-frog pass as two launches of the
 *                        single-stencil-field kernel (half A: v_{n+1}, u_{n+2} from P_v, S_u; half B:
 *                        v_{n+2}, u_{n+3} from S_v, U -- the two share no value), 64 x 32 tiles,
 *                        one register queue per CTA (default 1; 0 = the coupled pair kernel;
 *                        peer pushes always use the coupled kernel)
 *   "half_fe"      1/0   the forward-Euler substep through the same kernel (default 0)
 *   "fea"          1/0   sequences with n_k >= 4 on that path: the forward-Euler substep fused with
 *                        the first step of the u_1 leap-frog chain in one two-field pass (u_0, v_0 in;
 *                        v_1, u_2, v_2, u_3 out: 48 B per point instead of 40 + 32), lap(u_1) formed
 *                        as lap(u_0) + h lap(v_0) -- a rounding-level change; default 1)
 *   "fea_ring"     1/0   that fused pass with both stencil fields fed through rings of tiles (the
 *                        queue fronts read from the ring, not loaded again; bit-identical; default 1)
 *   "fin_ring"     1/0   the same for the LF + final pass (2 stages fit; measured slower, default 0)
 *   "half_tall"    1/0   64 x 32 tiles for the half kernel when ny % 32 == 0 (default 1)
 *   "half_rpt"     2/4   rows per thread of the tall half kernel (16 or 8 warps; default 4)
 *   "zchunk_fin"   k     planes per CTA of the LF + final pass only (0 = as the pair; default 0)
 *   "l2hint_fin"   bits  the LF + final pass's L2 policy bits (as "l2hint"; default 11)
 *   "streams"      1/2   sequences alternating over two CUDA streams on single-substep paths with
 *                        spare level buffers (2-D TMA grids, 3-D with fuse 0); final passes kept in
 *                        ascending n_k order by events, bit-identical (default 1: measured no faster)
 *   "l2hint_half"  bits  half kernel: 1 centre boxes evict_last, 2 streaming loads of the
 *                        pointwise field, 4 halo boxes evict_first, 8 streaming stores (default 11)
 *   "fuse2d"       1/0   2-D acoustics: two substeps per pass as the chain-U / chain-P
 *                        kernel pair (default 0: bit-identical but measured slower
 *                        than single substeps on B200)
 *   "persistent"   1/0   1-D grids up to 7000 points with m <= 16: every macro step of
 *                        a gbs_advance in one thread-block-cluster launch (default 1)
 *   "zchunk"       k     planes per CTA along the slowest axis (0 = automatic)
 *   "zchunk_pair"  k     the same for the two-substep 3-D kernel only (0 = "zchunk" if set,
 *                        else 256 when that leaves >= 8 waves of CTAs, otherwise 128)
 *   "band"         b     3-D TMA kernels: launch the x-y tiles in bands of b x-tiles (x fastest
 *                        inside a band); 0 or a b that does not divide the x-tile count =
 *                        whole rows (default 0; results do not depend on it)
 *   "l2hint"       bits  two-substep 3-D kernel L2 policies: 1 z+R centre boxes evict_last,
 *                        2 own-point boxes evict_first, 4 tile boxes evict_first, 8 streaming
 *                        stores (default 11; results do not depend on it)
 *   "l2hint_step"  bits  the same for the single-substep 3-D TMA kernel (1 = tile boxes
 *                        evict_last; default 0)
 *   "fused_combine" 1/0  sequence groups of the local transport: the fused combine above
 *                        (default 0: Comm all-reduce)
 *   "peer"         1/0   loopback slabs of a 3-D TMA grid: face planes pushed into the
 *                        neighbouring slabs' ghost planes by the producing kernels, ordered
 *                        by epoch flags (gbs_bind_peers), no halo exchange (default 0)
 *   "loopback_nccl" 1/0  loopback slabs exchange their ghost planes with grouped ncclSend /
 *                        ncclRecv on a one-rank communicator (the multi-GPU transfer path on one
 *                        GPU; graphs off, as with world > 1; default 0)
 *   "overlap"      1/0   slabbed layouts: exchange the ghost planes on a comm stream
 *                        while the interior planes are computed, then the face bands
 *                        (default 1)  */
GBS_API int gbs_set_option(gbs_ctx* ctx, const char* key, int64_t value);

/* Accumulated device time (ms) and launch count of the timed kernels of a class
 * since the last reset: cls 0 = interior LF, 1 = FE, 2 = final (average + weighted
 * accumulate), 3 = two LF substeps in one pass, 4 = LF + final in one pass, 5 = the
 * whole-run cluster kernel, 6 = one single-stencil-field half of a two-substep pass
 * (option "half"), 7 = the forward Euler fused with the first chain step (option "fea").
 * reset = 1 clears the counters after reading. */
GBS_API int gbs_kernel_time(gbs_ctx* ctx, int cls, double* total_ms, int64_t* launches, int reset);

GBS_API const char* gbs_strerror(int code);
GBS_API const char* gbs_last_error(const gbs_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* GBS_B200_H */

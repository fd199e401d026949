// gbs_exec.cu -- the schedule of one macro step (Eq. (1), lines 85-98,
// and the combination at lines 109-115, 221-225), per local slab:
//   for each sequence k of this rank's group, ascending n_k, h = H / n_k:
//     FE, n_k leap-frog steps, the final step fused with the averaging and the
//     weighted accumulate -- single-substep launches, or (3-D TMA grids) FE and
//     n_k/2 two-substep launches
//   [multi-GPU] ACC <- sum over sequence groups        (ncclAllReduce, fp64 sum)
//   swap(Y, ACC)
// On slabbed layouts the ghost planes of every stencil operand are refreshed
// before each launch (device copies between local slabs in loopback mode,
// ncclSend/ncclRecv between ranks), overlapped with the interior planes.
// gbs_advance replays the macro step as a CUDA graph.
#include "gbs_internal.h"
#include "gbs_wave3d_tma.cuh"     // substep modes and the TMA tile (no launches here)
#include "gbs_acoustic2d_pair.cuh"  // AC2_BH (band rows of the 2-D chain kernels)
#include "gbs_wave3d_half.cuh"      // HALF_LF / HALF_FE
#include "gbs_wave3d_pair.cuh"      // MODE_FEA

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
    if (c->slabs == 1 && c->loop_nccl) {
        // all slabs local, moved by NCCL point-to-point on a one-rank communicator (option
        // "loopback_nccl": the multi-GPU transfer path -- grouped ncclSend / ncclRecv straight
        // into the ghost planes, on the comm stream under overlap -- exercised on one GPU).
        // Every operation has peer 0, and NCCL pairs sends and receives to one peer in
        // posting order, so the receives are posted in the order of their matching sends.
        Comm* K = c->comm_slab;
        int rc;
        if ((rc = K->group_start(c))) return rc;
        for (int v = 0; v < nloc; ++v)
            for (int f : fields) {
                double* base = field_ptr(c, c->slab[v], b, f);
                if ((rc = K->send(c, base + (c->slab[v].nz - G) * P, cnt, 0, st))) return rc;   // up
                if ((rc = K->send(c, base, cnt, 0, st))) return rc;                             // down
            }
        for (int v = 0; v < nloc; ++v)
            for (int f : fields) {
                Slab& up = c->slab[(v + 1) % nloc];
                Slab& dn = c->slab[(v - 1 + nloc) % nloc];
                if ((rc = K->recv(c, field_ptr(c, up, b, f) - G * P, cnt, 0, st))) return rc;
                if ((rc = K->recv(c, field_ptr(c, dn, b, f) + dn.nz * P, cnt, 0, st))) return rc;
            }
        return K->group_end(c, st);
    }
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
    Slab& me = c->slab[0];
    unsigned fm = 0;
    for (int f : fields) fm |= 1u << f;
    const std::vector<gbs_halo_op> ops = halo_schedule(c->slabs, c->my_slab, me.nz, (int)G, fm);
    Comm* K = c->comm_slab;
    int rc;
    if ((rc = K->group_start(c))) return rc;
    for (const auto& op : ops) {
        double* p = field_ptr(c, me, b, op.field) + op.plane0 * P;
        const size_t n = (size_t)(op.planes * P);
        rc = op.kind == 0 ? K->send(c, p, n, op.peer, st) : K->recv(c, p, n, op.peer, st);
        if (rc) return rc;
    }
    return K->group_end(c, st);
}

// ---------------------------------------------------------------------------
// timing instrumentation (event pairs on the context stream)
// ---------------------------------------------------------------------------
int timed_begin(gbs_ctx* c, int cls, cudaEvent_t* end_ev) {
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
// `rows` > 0: the launch works in bands of that many rows (the 2-D chain kernels).
static int64_t face_band(const gbs_ctx* c, const Slab& s, int64_t rows) {
    if (rows > 0) return rows;
    if (c->pde == GBS_ACOUSTIC2D && c->use_bulk && s.tma_ok) return gbs::tma::TY;   // whole 16-row bands
    return c->R;
}

static bool overlap_halo(gbs_ctx* c, int64_t rows) {
    if (c->ghost == 0 || !c->use_overlap || c->slabs * c->loopback == 1) return false;
    for (const auto& s : c->slab)
        if (s.nz < 3 * face_band(c, s, rows)) return false;
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
static int run_overlapped(gbs_ctx* c, Launch&& launch, const std::vector<std::pair<int, unsigned>>& halos,
                          bool self_ghosts = false, int64_t rows = 0) {
    int rc;
    if (c->peer_on) {
        // peer pushes: no exchange -- each slab's launch stores its face planes into the
        // neighbours' ghost planes and waits (face CTAs only) for their previous launch;
        // then a one-thread kernel publishes this launch's epoch to both neighbours
        ++c->peer_epoch;
        for (size_t v = 0; v < c->slab.size(); ++v) {
            Slab& s = c->slab[v];
            if ((rc = launch(s, (int64_t)0, s.nz, (int64_t)0))) return rc;
            gbs::tma::peer_signal<<<1, 1, 0, c->stream>>>(peer_flag_remote(c, (int)v, 0),
                                                          peer_flag_remote(c, (int)v, 1), c->peer_epoch);
            c->launches++;
        }
        CU(c, cudaGetLastError());
        return GBS_OK;
    }
    if (c->ghost > 0 && c->slabs * c->loopback == 1) {
        // one slab with ghost rows (2-D TMA grids): only launches that read beyond the
        // slab (self_ghosts) need them, refreshed by one copy kernel; the rest wrap
        if (self_ghosts && (rc = launch_ghost_fill(c, halos))) return rc;
        return launch(c->slab[0], (int64_t)0, c->slab[0].nz, (int64_t)0);
    }
    if (!overlap_halo(c, rows)) {
        for (auto& h : halos)
            if ((rc = exchange_halo(c, h.first, h.second))) return rc;
        for (auto& s : c->slab)
            if ((rc = launch(s, (int64_t)0, s.nz, (int64_t)0))) return rc;
        return GBS_OK;
    }
    if ((rc = comm_fork(c))) return rc;
    for (auto& h : halos)
        if ((rc = exchange_halo(c, h.first, h.second, c->cstream))) return rc;
    for (auto& s : c->slab) {
        const int64_t B = face_band(c, s, rows);
        if ((rc = launch(s, B, s.nz - B, (int64_t)0))) return rc;      // interior: no ghosts read
    }
    // both face bands in one launch, queued on the comm stream behind the exchange: it starts
    // as soon as the ghosts are in and fills the SMs the interior launch's last wave leaves
    // idle (the two launches write disjoint planes; every in-place read is pointwise)
    std::swap(c->stream, c->cstream);                 // the launchers enqueue on c->stream
    for (auto& s : c->slab) {
        const int64_t B = face_band(c, s, rows);
        if ((rc = launch(s, (int64_t)0, s.nz, s.nz - 2 * B))) break;
    }
    std::swap(c->stream, c->cstream);
    if (rc) return rc;
    return comm_join(c);
}

static int step(gbs_ctx* c, int cls, const StepOperands& op) {
    int rc;
    cudaEvent_t end = nullptr;
    if (c->time_kernels && (rc = timed_begin(c, cls, &end))) return rc;
    rc = run_overlapped(c, [&](Slab& s, int64_t lo, int64_t hi, int64_t gap) { return launch_step(c, s, op, lo, hi, gap); },
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
    rc = run_overlapped(c, [&](Slab& s, int64_t lo, int64_t hi, int64_t gap) { return launch_pair(c, s, op, lo, hi, gap); },
                        {{op.Su.b, 1u << op.Su.f}, {op.U.b, 1u << op.U.f}});
    if (rc) return rc;
    if (end) CU(c, cudaEventRecord(end, c->stream));
    return GBS_OK;
}

// one single-stencil-field launch (gbs_wave3d_half.cuh): the halo of X is read
static int half_step(gbs_ctx* c, int cls, const HalfOperands& op) {
    int rc;
    cudaEvent_t end = nullptr;
    if (c->time_kernels && (rc = timed_begin(c, cls, &end))) return rc;
    rc = run_overlapped(c, [&](Slab& s, int64_t lo, int64_t hi, int64_t gap) { return launch_half(c, s, op, lo, hi, gap); },
                        {{op.X.b, 1u << op.X.f}});
    if (rc) return rc;
    if (end) CU(c, cudaEventRecord(end, c->stream));
    return GBS_OK;
}

// 2-D acoustics: two leap-frog substeps per pass (two chain kernels); they read S (p, u, v)
// and P (p, v) with y stencils
static int ac2d_pair_step(gbs_ctx* c, int cls, int P, int S, int Aout, int Bout, double cfA, double cfB) {
    int rc;
    cudaEvent_t end = nullptr;
    if (c->time_kernels && (rc = timed_begin(c, cls, &end))) return rc;
    rc = run_overlapped(
        c,
        [&](Slab& s, int64_t lo, int64_t hi, int64_t gap) {
            return launch_ac2d_pair(c, s, P, S, Aout, Bout, cfA, cfB, lo, hi, gap);
        },
        {{S, 0x7u}, {P, 0x5u}}, true, gbs::tma::AC2_BH);
    if (rc) return rc;
    if (end) CU(c, cudaEventRecord(end, c->stream));
    return GBS_OK;
}

// ---------------------------------------------------------------------------
// Fused combine across sequence groups (option "fused_combine"; PAPER.md:109-115,
// 398-400).  The slab's planes are split into g owner ranges, range j owned by group j.  The
// final pass of this group's last sequence is launched once per range j and stores its
// w-scaled partial sum straight into owner j's staging slot for this group (a store into the
// other context's memory: peer memory across GPUs, the same device here); after a fence every
// owner sums the g slots of its range in member order and stores the sum into every member's
// accumulator; a second fence and the accumulator is the next Y everywhere.  Same sums in the
// same order as the local transport's all-reduce: bit-identical to it.
// ---------------------------------------------------------------------------
static void owner_range(int64_t nz, int g, int j, int64_t* lo, int64_t* hi) {
    *lo = nz * j / g;
    *hi = nz * (j + 1) / g;
}

int64_t stage_bytes_of(const gbs_ctx* c) {
    int64_t mx = 0;
    const int64_t nz = c->nslow / std::max(1, c->slabs);
    for (int j = 0; j < c->groups; ++j) {
        int64_t lo, hi;
        owner_range(nz, c->groups, j, &lo, &hi);
        mx = std::max(mx, hi - lo);
    }
    return (int64_t)sizeof(double) * c->groups * c->F * mx * c->plane;
}

// member j's staging buffer and the base of its field f of buffer b (same layout on every member)
static double* member_stage(gbs_ctx* c, int j) {
    if (!c->grp_stage.empty()) return reinterpret_cast<double*>(c->grp_stage[j]);
    gbs_ctx* o = c->comm_group->member_ctx(j);
    return o ? o->d_stage : nullptr;
}
static double* member_field(gbs_ctx* c, int j, int b, int f) {
    double* mine = field_ptr(c, c->slab[0], b, f);
    if (!c->grp_ws.empty())
        return reinterpret_cast<double*>(c->grp_ws[j] + (reinterpret_cast<char*>(mine) - static_cast<char*>(c->ws_ptr)));
    gbs_ctx* o = c->comm_group->member_ctx(j);
    return o ? field_ptr(o, o->slab[0], b, f) : nullptr;
}

static int fused_final_pass(gbs_ctx* c, const PairOperands& fin) {
    const int g = c->groups, me = c->my_group, F = c->F;
    Slab& s = c->slab[0];
    const int64_t P = c->plane;
    int rc;
    if (c->grp_stage.empty() && !c->d_stage) {
        c->stage_doubles = stage_bytes_of(c) / (int64_t)sizeof(double);
        CU(c, cudaMalloc(&c->d_stage, sizeof(double) * (size_t)std::max<int64_t>(c->stage_doubles, 1)));
    }
    double* my_stage = member_stage(c, me);
    // the halos of the stencil operands, then the pass per owner range (no overlap split)
    if (c->ghost > 0 && c->slabs > 1) {
        if ((rc = exchange_halo(c, fin.Su.b, 1u << fin.Su.f))) return rc;
        if ((rc = exchange_halo(c, fin.U.b, 1u << fin.U.f))) return rc;
    }
    // every member has allocated its staging buffer and finished reading its previous ones
    if ((rc = c->comm_group->fence(c, c->stream))) return rc;
    for (int j = 0; j < g; ++j) {
        double* st = member_stage(c, j);
        if (!st) return fail(c, GBS_E_STATE, "fused combine: member %d has no staging buffer", j);
        int64_t lo, hi;
        owner_range(s.nz, g, j, &lo, &hi);
        if (hi <= lo) continue;
        PairOperands op = fin;
        // plane z of this slab lands at slot (me, f) of owner j, offset by its first plane
        op.out_u = st + ((int64_t)(me * F + 0) * (hi - lo) - lo) * P;
        op.out_v = st + ((int64_t)(me * F + 1) * (hi - lo) - lo) * P;
        if ((rc = launch_pair(c, s, op, lo, hi, 0))) return rc;
    }
    if ((rc = c->comm_group->fence(c, c->stream))) return rc;
    int64_t lo, hi;
    owner_range(s.nz, g, me, &lo, &hi);
    const int ACC = fin.Bu.b;
    for (int f = 0; f < F; ++f) {
        std::vector<double*> in(g), out(g);
        for (int i = 0; i < g; ++i) {
            in[i] = my_stage + (int64_t)(i * F + f) * (hi - lo) * P;
            double* acc = member_field(c, i, ACC, f);
            if (!acc) return fail(c, GBS_E_STATE, "fused combine: member %d's accumulator unknown", i);
            out[i] = acc + lo * P;
        }
        if ((rc = owner_combine(c, in.data(), out.data(), g, (hi - lo) * P, c->stream))) return rc;
    }
    return c->comm_group->fence(c, c->stream);
}

static bool fused_path(const gbs_ctx* c) {
    if (!(c->use_fuse && c->use_bulk && c->nbuf == 6)) return false;
    for (const auto& s : c->slab)
        if (!s.tma_ok) return false;
    return true;
}

int harvest_timer(gbs_ctx* c) {
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
    bool combined = false;            // the fused combine already summed the groups
    const bool fused = fused_path(c) && c->pde == GBS_WAVE3D;
    bool fused2d = fused_path(c) && c->use_fuse2d && c->pde == GBS_ACOUSTIC2D;
    for (const auto& s : c->slab)                  // the chain kernels work in whole 32-row bands
        if (s.nz % gbs::tma::AC2_BH) fused2d = false;
    // two sequence streams: single-substep paths on one slab with 6 state buffers (2-D TMA grids)
    const bool two = c->n_streams == 2 && !fused && !fused2d && c->nbuf >= 6 && c->slabs * c->loopback == 1 &&
                     !c->time_kernels && c->my_seq.size() > 1;
    if (two) {
        if (!c->stream2) {
            CU(c, cudaStreamCreateWithFlags(&c->stream2, cudaStreamNonBlocking));
            CU(c, cudaEventCreateWithFlags(&c->ev_fork2, cudaEventDisableTiming));
            CU(c, cudaEventCreateWithFlags(&c->ev_join2, cudaEventDisableTiming));
            CU(c, cudaEventCreateWithFlags(&c->ev_fin, cudaEventDisableTiming));
        }
        CU(c, cudaEventRecord(c->ev_fork2, c->stream));
        CU(c, cudaStreamWaitEvent(c->stream2, c->ev_fork2, 0));
    }
    for (size_t q = 0; q < c->my_seq.size(); ++q) {
        const int k = c->my_seq[q];
        const int n = c->nk_all[k];
        const double h = H / (double)n;
        const bool last = (q + 1 == c->my_seq.size());
        if (fused2d) {
            // FE and LF1 single, then (LF2, LF3), ..., (LF_{n-2}, LF_{n-1}) two per pass
            // (buffers (2,3) -> (4,5) -> (2,3) ...), then the final step single
            if ((rc = step(c, 1, {Y, Y, 2, gbs::MODE_FE, h, 0.0, false}))) return rc;        // y1
            if ((rc = step(c, 0, {2, Y, 3, gbs::MODE_LF, 2.0 * h, 0.0, false}))) return rc;  // y2
            int P = 2, S = 3;
            for (int p = 0; p < (n - 2) / 2; ++p) {
                const int A = P == 2 ? 4 : 2, B = A + 1;
                if ((rc = ac2d_pair_step(c, 3, P, S, A, B, 2.0 * h, 2.0 * h))) return rc;
                P = A; S = B;
            }
            StepOperands fin{S, P, ACC, first ? gbs::MODE_FIN0 : gbs::MODE_FINACC, h, 0.5 * c->wk_all[k], last};
            if ((rc = step(c, 2, fin))) return rc;
            first = false;
            continue;
        }
        if (fused) {
            // FE (which also forms u_2), then n/2 launches of two substeps:
            // (LF1, LF2), ..., (LF_{n-1}, final).  Field slots: y1 -> buffer 2; the
            // u-levels rotate through (2,0)/(3,0) and (4,0)/(5,0); v_{odd} stays in
            // (2,1) and v_{even} in (3,1), both updated in place (pointwise reads).
            const bool half = half_eligible(c);
            // FE fused with chain A's first step (option "fea"; gbs_wave3d_pair.cuh MODE_FEA)
            const bool fea = half && c->use_fea && n >= 4;
            if (fea) {
                PairOperands fe{Slot{Y, 1}, Slot{Y, 0}, Slot{Y, 1}, Slot{Y, 1},
                                Slot{3, 1}, Slot{4, 0}, Slot{2, 1}, Slot{3, 0},
                                gbs::tma::MODE_FEA, h, 2.0 * h, 0.0, false};
                if ((rc = pair_step(c, 7, fe))) return rc;     // v2, u3 | v1, u2
            } else if (half && c->half_fe) {
                // v1 = v0 + h lap(u0), u2 = u0 + 2h v1, u1 = u0 + h v0 (the FE kernel's values)
                HalfOperands fe{gbs::tma::HALF_FE, Slot{Y, 0}, Slot{Y, 1}, Slot{2, 1}, Slot{3, 0}, Slot{2, 0},
                                h, 2.0 * h};
                if ((rc = half_step(c, 1, fe))) return rc;
            } else {
                StepOperands fe{Y, Y, 2, gbs::MODE_FE, h, 0.0, false};
                fe.xu = Slot{3, 0};
                fe.cf2 = 2.0 * h;
                if ((rc = step(c, 1, fe))) return rc;                                        // y1, u2
            }
            Slot Pv{Y, 1}, Su{2, 0}, Sv{2, 1}, U{3, 0};
            for (int p = 0; p < n / 2; ++p) {
                if (p + 1 < n / 2) {
                    const int nb = Su.b == 2 ? 4 : 2;
                    PairOperands op{Pv, Su, Sv, U, Slot{3, 1}, Slot{nb, 0}, Sv, Slot{nb + 1, 0},
                                    gbs::MODE_LF, 2.0 * h, 2.0 * h, 0.0, false};
                    if (half) {
                        // the pair's two independent halves (gbs_wave3d_half.cuh): neither reads
                        // what the other writes
                        HalfOperands ha{gbs::tma::HALF_LF, op.Su, op.Pv, op.Av, op.Bu};
                        ha.c1 = op.cfA; ha.c2 = op.cfB;
                        HalfOperands hb{gbs::tma::HALF_LF, op.U, op.Sv, op.Bv, op.Cu};
                        hb.c1 = op.cfB; hb.c2 = op.cfA;
                        if (!(fea && p == 0) && (rc = half_step(c, 6, ha))) return rc;   // FEA did A0
                        if ((rc = half_step(c, 6, hb))) return rc;
                    } else if ((rc = pair_step(c, 3, op))) {
                        return rc;
                    }
                    Pv = Slot{3, 1}; Su = Slot{nb, 0}; U = Slot{nb + 1, 0};
                } else {
                    PairOperands fin{Pv, Su, Sv, U, Slot{ACC, 0}, Slot{ACC, 0}, Slot{ACC, 1}, Slot{ACC, 0},
                                     first ? gbs::MODE_FIN0 : gbs::MODE_FINACC, 2.0 * h, h,
                                     0.5 * c->wk_all[k], last};
                    if (last && c->fused_combine && c->groups > 1) {
                        if ((rc = fused_final_pass(c, fin))) return rc;
                        combined = true;
                    } else if ((rc = pair_step(c, 4, fin))) {
                        return rc;
                    }
                }
            }
            first = false;
            continue;
        }
        // two streams (option "streams"): sequence q on stream q % 2 with its own level buffers
        // ({2,3} or {4,5}); the final passes stay in ascending n_k order (each waits for the
        // previous one's event), so the accumulation order -- and the result -- is unchanged
        const bool alt = two && (q % 2 == 1);
        const int b1 = alt ? 4 : B, b2 = alt ? 5 : C;
        cudaStream_t main_stream = c->stream;
        if (alt) c->stream = c->stream2;
        if ((rc = step(c, 1, {Y, Y, b1, gbs::MODE_FE, h, 0.0, false}))) { c->stream = main_stream; return rc; }
        if ((rc = step(c, 0, {b1, Y, b2, gbs::MODE_LF, 2.0 * h, 0.0, false}))) { c->stream = main_stream; return rc; }
        int prev = b1, cur = b2;
        for (int i = 2; i <= n - 1; ++i) {                                                    // y3..yN
            if ((rc = step(c, 0, {cur, prev, prev, gbs::MODE_LF, 2.0 * h, 0.0, false}))) { c->stream = main_stream; return rc; }
            std::swap(prev, cur);
        }
        StepOperands fin{cur, prev, ACC, first ? gbs::MODE_FIN0 : gbs::MODE_FINACC, h,
                         0.5 * c->wk_all[k], last};
        if (two && !first) {
            cudaError_t e = cudaStreamWaitEvent(c->stream, c->ev_fin, 0);
            if (e != cudaSuccess) { c->stream = main_stream; return fail(c, GBS_E_CUDA, "stream wait: %s", cudaGetErrorString(e)); }
        }
        rc = step(c, 2, fin);
        if (!rc && two) {
            cudaError_t e = cudaEventRecord(c->ev_fin, c->stream);
            if (e != cudaSuccess) rc = fail(c, GBS_E_CUDA, "event record: %s", cudaGetErrorString(e));
        }
        c->stream = main_stream;
        if (rc) return rc;
        first = false;
    }
    if (two) {
        // join the second stream (its last final pass precedes the main stream's, or is it)
        CU(c, cudaEventRecord(c->ev_join2, c->stream2));
        CU(c, cudaStreamWaitEvent(c->stream, c->ev_join2, 0));
    }
    if (c->groups > 1 && !combined) {
        // Y <- sum over the sequence groups of their w-scaled partial sums
        Slab& s = c->slab[0];
        double* p[3];
        size_t n[3];
        for (int f = 0; f < c->F; ++f) {
            p[f] = field_ptr(c, s, ACC, f);
            n[f] = (size_t)(s.nz * c->plane);
        }
        if ((rc = c->comm_group->allreduce_sum(c, p, n, c->F, c->stream))) return rc;
    }
    c->yb = ACC;
    c->launches_per_macro = c->launches - l0;
    return GBS_OK;
}

extern "C" {

static int advance_impl(gbs_ctx* c, int64_t macro_steps, double H);

// a rank of the local transport that fails wakes the members waiting for it in a collective
int gbs_advance(gbs_ctx* c, int64_t macro_steps, double H) {
    if (!c) return fail(c, GBS_E_INVAL, "ctx is NULL");
    return comm_abort_on_error(c, advance_impl(c, macro_steps, H));
}

}  // extern "C"

static int advance_impl(gbs_ctx* c, int64_t macro_steps, double H) {
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
    if (c->peer_on) {
        if (!peer_eligible(c, c->world > 1) || !fused_path(c))
            return fail(c, GBS_E_UNSUPPORTED, "peer halo pushes need the slabbed 3-D two-substep path");
        if (!c->peer_ghosts_valid) {
            // a freshly written state: fill Y's ghost planes once by the ordinary exchange; from
            // then on every macro step's final kernels push them
            int rc2 = exchange_halo(c, c->yb, 0x1u);
            if (rc2) return rc2;
            c->peer_ghosts_valid = true;
        }
    }
    const bool graph = c->use_graph && !c->time_kernels && !c->peer_on && macro_steps > 0;
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

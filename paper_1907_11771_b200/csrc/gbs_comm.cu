// gbs_comm.cu -- the collectives of the macro step behind one
// interface (gbs_internal.h, struct Comm), with two transports:
//
//   NCCL   one process per GPU (the production path): ncclCommInitRank from the
//          caller's unique id, ncclCommSplit into the slab and group
//          communicators, grouped ncclSend/ncclRecv for the halo planes,
//          ncclAllReduce(sum, fp64) for the combine across sequence groups
//          ("combined after the barrier"; §3.6, 388-400) and
//          ncclAllGather for gbs_read_state.
//   local  every rank is a context of THIS process on one device, driven by its
//          own host thread (gbs_local_hub_create; the tests' multi-rank harness).
//          The same call sites run with device-to-device copies ordered by
//          events and host barriers, so gbs_create's split, the plan, the halo
//          schedule, the group combine and the gather execute exactly as they do
//          on N GPUs.  No kernel ever waits on another rank's kernel (every
//          cross-rank dependency is a stream-ordered event wait that the host
//          enqueues only after the producer's record), so the emulation is safe
//          on one GPU (B200_PROFILING.md: "do not run kernels that wait on one
//          another as separate launches").
//
// Semantics of the local transport (a rendezvous, like NCCL's blocking p2p):
//   group_end  record READY on the stream; barrier; each rank waits for the
//              READY of every peer it receives from and copies, in posting order
//              per peer pair, the k-th send of peer p to it into its k-th receive
//              from p (NCCL's matching rule); record DONE; barrier; each rank
//              waits for the DONE of every peer it sent to (the sources may be
//              overwritten only after they were read).
//   allreduce  (in place, sum) READY; barrier; rank i launches one kernel that,
//              for its 1/n share of the elements, sums the n members' buffers in
//              member order (fixed, deterministic) and stores the sum into every
//              member's buffer -- reduce-scatter and all-gather in one pass;
//              DONE; barrier; wait for every member's DONE.
//   allgather  READY; barrier; copy every member's block into dst; DONE;
//              barrier; wait for every member's DONE.
#include "gbs_internal.h"

#include <chrono>
#include <condition_variable>
#include <map>
#include <memory>
#include <mutex>

// ---------------------------------------------------------------------------
// NCCL transport
// ---------------------------------------------------------------------------
namespace {

struct NcclComm final : Comm {
    nccl::comm_t h = nullptr;
    explicit NcclComm(nccl::comm_t c, int r, int n) : h(c) { rank = r; size = n; }
    ~NcclComm() override {
        auto& A = nccl::api();
        if (h && A.ok) A.CommDestroy(h);
    }
    bool is_nccl() const override { return true; }
    int group_start(gbs_ctx* c) override {
        NC(c, nccl::api().GroupStart());
        return GBS_OK;
    }
    int send(gbs_ctx* c, const double* p, size_t n, int peer, cudaStream_t st) override {
        NC(c, nccl::api().Send(p, n, nccl::ncclFloat64, peer, h, st));
        return GBS_OK;
    }
    int recv(gbs_ctx* c, double* p, size_t n, int peer, cudaStream_t st) override {
        NC(c, nccl::api().Recv(p, n, nccl::ncclFloat64, peer, h, st));
        return GBS_OK;
    }
    int group_end(gbs_ctx* c, cudaStream_t) override {
        NC(c, nccl::api().GroupEnd());
        return GBS_OK;
    }
    int allreduce_sum(gbs_ctx* c, double* const* p, const size_t* n, int k, cudaStream_t st) override {
        auto& A = nccl::api();
        NC(c, A.GroupStart());
        for (int i = 0; i < k; ++i) NC(c, A.AllReduce(p[i], p[i], n[i], nccl::ncclFloat64, nccl::ncclSum, h, st));
        NC(c, A.GroupEnd());
        return GBS_OK;
    }
    int allgather(gbs_ctx* c, const double* src, double* dst, size_t n, cudaStream_t st) override {
        NC(c, nccl::api().AllGather(src, dst, n, nccl::ncclFloat64, h, st));
        return GBS_OK;
    }
    int fence(gbs_ctx* c, cudaStream_t st) override {
        if (!c->d_fence) CU(c, cudaMalloc(&c->d_fence, sizeof(double)));
        NC(c, nccl::api().AllReduce(c->d_fence, c->d_fence, 1, nccl::ncclFloat64, nccl::ncclSum, h, st));
        return GBS_OK;
    }
    int split(gbs_ctx* c, int color, int key, Comm** out) override {
        nccl::comm_t s = nullptr;
        int r = nccl::api().CommSplit(h, color, key, &s, nullptr);
        if (r) return fail(c, GBS_E_NCCL, "ncclCommSplit: %s", nccl::api().GetErrorString(r));
        // rank / size inside the new communicator: filled by the caller (it knows the plan)
        *out = new NcclComm(s, 0, 1);
        return GBS_OK;
    }
};

// ---------------------------------------------------------------------------
// local transport
// ---------------------------------------------------------------------------
constexpr int kMaxMembers = 64;

struct SumPtrs {
    double* p[kMaxMembers];
};

// out_j[e] = sum_{i=0..n-1} in_i[e] (member order) for e in [e0, e1), stored into every member
__global__ void local_sum_kernel(SumPtrs P, int n, int64_t e0, int64_t e1) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t e = e0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < e1; e += stride) {
        double s = P.p[0][e];
        for (int i = 1; i < n; ++i) s += P.p[i][e];
        for (int i = 0; i < n; ++i) P.p[i][e] = s;
    }
}

}  // namespace

// the fused combine's owner step: out_j[e] = sum_i in_i[e] (member order) for every member j
__global__ void owner_combine_kernel(SumPtrs in, SumPtrs out, int n, int64_t count) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < count; e += stride) {
        double s = in.p[0][e];
        for (int i = 1; i < n; ++i) s += in.p[i][e];
        for (int j = 0; j < n; ++j) out.p[j][e] = s;
    }
}

int owner_combine(gbs_ctx* c, double* const* in, double* const* out, int n, int64_t count, cudaStream_t st) {
    if (n > kMaxMembers) return fail(c, GBS_E_UNSUPPORTED, "fused combine: > %d groups", kMaxMembers);
    if (count <= 0) return GBS_OK;
    SumPtrs I{}, O{};
    for (int i = 0; i < n; ++i) { I.p[i] = in[i]; O.p[i] = out[i]; }
    const int64_t blocks = std::min<int64_t>((count + 255) / 256, (int64_t)c->sms * 8);
    owner_combine_kernel<<<(unsigned)blocks, 256, 0, st>>>(I, O, n, count);
    CU(c, cudaGetLastError());
    c->launches++;
    return GBS_OK;
}

namespace {

struct Posted {
    int kind;            // 0 send, 1 recv
    int peer;
    double* ptr;
    size_t n;
};

// State shared by the members of one communicator (the world of a hub, or one split color).
struct Shared {
    int n = 0;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    uint64_t gen = 0;
    int device = 0;
    std::vector<cudaEvent_t> ready, done;     // per member
    std::vector<std::vector<Posted>> posted;  // per member (p2p groups)
    std::vector<std::vector<double*>> bufs;   // per member (allreduce / allgather arguments)
    std::vector<std::vector<size_t>> counts;
    std::vector<gbs_ctx*> ctx;                // per member (local transport: same process)
    std::vector<std::pair<int, int>> split_in;                          // (color, key) per member
    std::vector<std::pair<std::shared_ptr<Shared>, int>> split_out;    // (communicator, rank)
    bool broken = false;

    explicit Shared(int n_, int dev) : n(n_), device(dev), ready(n_, nullptr), done(n_, nullptr),
                                       posted(n_), bufs(n_), counts(n_), ctx(n_, nullptr), split_in(n_),
                                       split_out(n_) {}
    ~Shared() {
        for (auto e : ready) if (e) cudaEventDestroy(e);
        for (auto e : done) if (e) cudaEventDestroy(e);
    }
    // generation barrier; a member that never arrives fails everyone after the timeout
    bool barrier() {
        std::unique_lock<std::mutex> lk(mu);
        if (broken) return false;
        const uint64_t g = gen;
        if (++arrived == n) {
            arrived = 0;
            ++gen;
            cv.notify_all();
            return true;
        }
        const bool ok = cv.wait_for(lk, std::chrono::seconds(300), [&] { return gen != g || broken; });
        if (!ok || broken) {
            broken = true;
            cv.notify_all();
            return false;
        }
        return true;
    }
};

struct LocalHub {
    int world;
    std::shared_ptr<Shared> shared;
};

struct LocalComm final : Comm {
    std::shared_ptr<Shared> S;
    std::vector<Posted> pend;
    LocalComm(std::shared_ptr<Shared> s, int r) : S(std::move(s)) { rank = r; size = S->n; }
    bool is_nccl() const override { return false; }

    int ev_init(gbs_ctx* c) {
        if (S->ready[rank]) return GBS_OK;
        CU(c, cudaEventCreateWithFlags(&S->ready[rank], cudaEventDisableTiming));
        CU(c, cudaEventCreateWithFlags(&S->done[rank], cudaEventDisableTiming));
        return GBS_OK;
    }
    int bar(gbs_ctx* c) {
        if (!S->barrier())
            return fail(c, GBS_E_NCCL, "local transport: a member rank failed or did not reach the collective (300 s)");
        return GBS_OK;
    }
    int group_start(gbs_ctx*) override {
        pend.clear();
        return GBS_OK;
    }
    int send(gbs_ctx*, const double* p, size_t n, int peer, cudaStream_t) override {
        pend.push_back({0, peer, const_cast<double*>(p), n});
        return GBS_OK;
    }
    int recv(gbs_ctx*, double* p, size_t n, int peer, cudaStream_t) override {
        pend.push_back({1, peer, p, n});
        return GBS_OK;
    }
    int group_end(gbs_ctx* c, cudaStream_t st) override {
        int rc;
        if ((rc = ev_init(c))) return rc;
        S->posted[rank] = pend;
        CU(c, cudaEventRecord(S->ready[rank], st));
        if ((rc = bar(c))) return rc;
        // match my receives with the peers' sends to me, per peer in posting order
        std::vector<int> used(size, 0);
        std::vector<char> waited(size, 0);
        for (const Posted& r : pend) {
            if (r.kind != 1) continue;
            if (r.peer < 0 || r.peer >= size) return fail(c, GBS_E_NCCL, "local transport: recv peer %d", r.peer);
            const std::vector<Posted>& ps = S->posted[r.peer];
            int k = used[r.peer]++, seen = 0;
            const Posted* m = nullptr;
            for (const Posted& s : ps)
                if (s.kind == 0 && s.peer == rank && seen++ == k) { m = &s; break; }
            if (!m) return fail(c, GBS_E_NCCL, "local transport: receive %d from %d has no matching send", k, r.peer);
            if (m->n != r.n)
                return fail(c, GBS_E_NCCL, "local transport: send of %zu values matched a receive of %zu", m->n, r.n);
            if (!waited[r.peer]) {
                CU(c, cudaStreamWaitEvent(st, S->ready[r.peer], 0));
                waited[r.peer] = 1;
            }
            CU(c, cudaMemcpyAsync(r.ptr, m->ptr, r.n * sizeof(double), cudaMemcpyDeviceToDevice, st));
        }
        // every send of mine must have been received (NCCL would hang otherwise)
        for (int p = 0; p < size; ++p) {
            int sends = 0, recvs = 0;
            for (const Posted& s : pend) sends += (s.kind == 0 && s.peer == p);
            for (const Posted& r : S->posted[p]) recvs += (r.kind == 1 && r.peer == rank);
            if (sends != recvs)
                return fail(c, GBS_E_NCCL, "local transport: %d sends to %d but it posted %d receives", sends, p, recvs);
        }
        CU(c, cudaEventRecord(S->done[rank], st));
        if ((rc = bar(c))) return rc;
        std::vector<char> w(size, 0);
        for (const Posted& s : pend)
            if (s.kind == 0 && !w[s.peer]) {
                CU(c, cudaStreamWaitEvent(st, S->done[s.peer], 0));
                w[s.peer] = 1;
            }
        pend.clear();
        return GBS_OK;
    }
    int allreduce_sum(gbs_ctx* c, double* const* p, const size_t* n, int k, cudaStream_t st) override {
        int rc;
        if ((rc = ev_init(c))) return rc;
        if (size > kMaxMembers) return fail(c, GBS_E_UNSUPPORTED, "local transport: > %d members", kMaxMembers);
        S->bufs[rank].assign(p, p + k);
        S->counts[rank].assign(n, n + k);
        CU(c, cudaEventRecord(S->ready[rank], st));
        if ((rc = bar(c))) return rc;
        for (int j = 0; j < size; ++j) {
            if (S->bufs[j].size() != (size_t)k) return fail(c, GBS_E_NCCL, "local allreduce: buffer count mismatch");
            for (int i = 0; i < k; ++i)
                if (S->counts[j][i] != n[i]) return fail(c, GBS_E_NCCL, "local allreduce: count mismatch");
            if (j != rank) CU(c, cudaStreamWaitEvent(st, S->ready[j], 0));
        }
        for (int i = 0; i < k; ++i) {
            SumPtrs P{};
            for (int j = 0; j < size; ++j) P.p[j] = S->bufs[j][i];
            const int64_t e0 = (int64_t)(n[i] * rank / size), e1 = (int64_t)(n[i] * (rank + 1) / size);
            if (e1 > e0) {
                const int64_t blocks = std::min<int64_t>((e1 - e0 + 255) / 256, (int64_t)c->sms * 8);
                local_sum_kernel<<<(unsigned)blocks, 256, 0, st>>>(P, size, e0, e1);
                CU(c, cudaGetLastError());
                c->launches++;
            }
        }
        CU(c, cudaEventRecord(S->done[rank], st));
        if ((rc = bar(c))) return rc;
        for (int j = 0; j < size; ++j)
            if (j != rank) CU(c, cudaStreamWaitEvent(st, S->done[j], 0));
        return GBS_OK;
    }
    int allgather(gbs_ctx* c, const double* src, double* dst, size_t n, cudaStream_t st) override {
        int rc;
        if ((rc = ev_init(c))) return rc;
        S->bufs[rank].assign(1, const_cast<double*>(src));
        S->counts[rank].assign(1, n);
        CU(c, cudaEventRecord(S->ready[rank], st));
        if ((rc = bar(c))) return rc;
        for (int j = 0; j < size; ++j) {
            if (S->counts[j].size() != 1 || S->counts[j][0] != n)
                return fail(c, GBS_E_NCCL, "local allgather: count mismatch");
            if (j != rank) CU(c, cudaStreamWaitEvent(st, S->ready[j], 0));
            CU(c, cudaMemcpyAsync(dst + (size_t)j * n, S->bufs[j][0], n * sizeof(double), cudaMemcpyDeviceToDevice, st));
        }
        CU(c, cudaEventRecord(S->done[rank], st));
        if ((rc = bar(c))) return rc;
        for (int j = 0; j < size; ++j)
            if (j != rank) CU(c, cudaStreamWaitEvent(st, S->done[j], 0));
        return GBS_OK;
    }
    int fence(gbs_ctx* c, cudaStream_t st) override {
        int rc;
        if ((rc = ev_init(c))) return rc;
        CU(c, cudaEventRecord(S->ready[rank], st));
        if ((rc = bar(c))) return rc;
        for (int j = 0; j < size; ++j)
            if (j != rank) CU(c, cudaStreamWaitEvent(st, S->ready[j], 0));
        // nobody records READY again before every member has enqueued its waits
        return bar(c);
    }
    gbs_ctx* member_ctx(int i) override { return (i >= 0 && i < size) ? S->ctx[i] : nullptr; }
    void abort() override {
        std::lock_guard<std::mutex> lk(S->mu);
        S->broken = true;
        S->cv.notify_all();
    }
    void register_ctx(gbs_ctx* c) override { S->ctx[rank] = c; }
    int split(gbs_ctx* c, int color, int key, Comm** out) override {
        int rc;
        S->split_in[rank] = {color, key};
        if ((rc = bar(c))) return rc;
        if (rank == 0) {
            std::map<int, std::vector<std::pair<int, int>>> by;      // color -> (key, member)
            for (int j = 0; j < size; ++j) by[S->split_in[j].first].push_back({S->split_in[j].second, j});
            for (auto& kv : by) {
                std::sort(kv.second.begin(), kv.second.end());
                auto sh = std::make_shared<Shared>((int)kv.second.size(), S->device);
                for (size_t r = 0; r < kv.second.size(); ++r) S->split_out[kv.second[r].second] = {sh, (int)r};
            }
        }
        if ((rc = bar(c))) return rc;
        auto res = S->split_out[rank];
        if ((rc = bar(c))) return rc;            // everyone has taken its result
        S->split_out[rank] = {nullptr, 0};
        *out = new LocalComm(res.first, res.second);
        return GBS_OK;
    }
};

}  // namespace

// ---------------------------------------------------------------------------
// communicator setup for gbs_create (world > 1)
// ---------------------------------------------------------------------------
int comm_init(gbs_ctx* c, const gbs_dist* d) {
    if (d->transport == GBS_TRANSPORT_LOCAL) {
        auto* hub = static_cast<LocalHub*>(d->hub);
        if (!hub) return fail(c, GBS_E_INVAL, "dist.transport = GBS_TRANSPORT_LOCAL needs dist.hub");
        if (hub->world != c->world) return fail(c, GBS_E_INVAL, "hub of %d ranks, dist.world = %d", hub->world, c->world);
        if (hub->shared->device != c->device)
            return fail(c, GBS_E_INVAL, "local transport: every rank must use device %d", hub->shared->device);
        c->comm_world = new LocalComm(hub->shared, c->rank);
        c->local_transport = true;
    } else if (d->transport == GBS_TRANSPORT_NCCL) {
        auto& A = nccl::api();
        if (!A.ok) return fail(c, GBS_E_NCCL, "libnccl.so.2 not found");
        nccl::uid_t id;
        memcpy(&id, d->nccl_id, 128);
        nccl::comm_t w = nullptr;
        int r = A.CommInitRank(&w, c->world, id, c->rank);
        if (r) return fail(c, GBS_E_NCCL, "ncclCommInitRank: %s", A.GetErrorString(r));
        c->comm_world = new NcclComm(w, c->rank, c->world);
    } else {
        return fail(c, GBS_E_INVAL, "dist.transport=%d", d->transport);
    }
    int rc;
    // every rank takes part in both splits (collective over the world), as ncclCommSplit requires
    Comm* s = nullptr;
    Comm* g = nullptr;
    if ((rc = c->comm_world->split(c, c->my_group, c->my_slab, &s))) return rc;
    if ((rc = c->comm_world->split(c, c->my_slab, c->my_group, &g))) { delete s; return rc; }
    s->rank = c->my_slab; s->size = c->slabs;
    g->rank = c->my_group; g->size = c->groups;
    c->comm_slab = s;
    c->comm_group = g;
    c->comm_group->register_ctx(c);
    return GBS_OK;
}

// one-rank NCCL communicator for option "loopback_nccl"
int comm_nccl_self(gbs_ctx* c, Comm** out) {
    auto& A = nccl::api();
    if (!A.ok) return fail(c, GBS_E_NCCL, "libnccl.so.2 not found");
    nccl::uid_t id;
    nccl::comm_t h = nullptr;
    int r = A.GetUniqueId(&id);
    if (!r) r = A.CommInitRank(&h, 1, id, 0);
    if (r) return fail(c, GBS_E_NCCL, "one-rank communicator: %s", A.GetErrorString(r));
    *out = new NcclComm(h, 0, 1);
    return GBS_OK;
}

int comm_abort_on_error(gbs_ctx* c, int rc) {
    if (rc != GBS_OK && c && c->local_transport)
        for (Comm* k : {c->comm_world, c->comm_slab, c->comm_group})
            if (k) k->abort();
    return rc;
}

void comm_release(gbs_ctx* c) {
    delete c->comm_group;
    delete c->comm_slab;
    delete c->comm_world;
    c->comm_group = c->comm_slab = c->comm_world = nullptr;
}

extern "C" {

int gbs_local_hub_create(int world, int device, void** hub) {
    if (!hub) return fail(nullptr, GBS_E_INVAL, "hub is NULL");
    *hub = nullptr;
    if (world < 1 || world > kMaxMembers) return fail(nullptr, GBS_E_INVAL, "world=%d (1..%d)", world, kMaxMembers);
    auto* h = new (std::nothrow) LocalHub();
    if (!h) return fail(nullptr, GBS_E_NOMEM, "host allocation failed");
    h->world = world;
    h->shared = std::make_shared<Shared>(world, device);
    *hub = h;
    return GBS_OK;
}

void gbs_local_hub_destroy(void* hub) { delete static_cast<LocalHub*>(hub); }

}  // extern "C"

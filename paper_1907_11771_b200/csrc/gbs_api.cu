// gbs_api.cu -- the C ABI surface (include/gbs.h): context creation (validate,
// plan, allocate, join NCCL), options, queries, error strings, destruction.
// The rest of the library: gbs_plan.cu, gbs_launch.cu, gbs_exec.cu, gbs_io.cu
// (gbs_internal.h).
#include "gbs_internal.h"

namespace nccl {
// NCCL, resolved at run time from the process (torch's libnccl.so.2) so the
// library loads on machines without NCCL and never links a second copy.
Api& api() {
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

namespace cufft {
Api& api() {
    static Api a;
    static bool tried = false;
    if (tried) return a;
    tried = true;
    void* h = dlopen("libcufft.so.11", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libcufft.so.11", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libcufft.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return a;
#define CUFFT_SYM(name) a.name = (decltype(a.name))dlsym(h, "cufft" #name); if (!a.name) return a;
    CUFFT_SYM(Plan1d) CUFFT_SYM(ExecD2Z) CUFFT_SYM(ExecZ2D) CUFFT_SYM(SetStream) CUFFT_SYM(Destroy)
#undef CUFFT_SYM
    a.ok = true;
    return a;
}
}  // namespace cufft

thread_local std::string g_err;

int fail(gbs_ctx* c, int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    if (c) c->err = buf;
    g_err = buf;
    return code;
}

static int build_ctx(gbs_ctx* c) { return alloc_state(c); }

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
    if (c->stream2) { cudaStreamSynchronize(c->stream2); cudaStreamDestroy(c->stream2); }
    for (cudaEvent_t e : {c->ev_fork2, c->ev_join2, c->ev_fin})
        if (e) cudaEventDestroy(e);
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
    if (c->d_peer_flags) cudaFree(c->d_peer_flags);
    if (c->d_stage) cudaFree(c->d_stage);
    if (c->d_fence) cudaFree(c->d_fence);
    spectral_release(c);
    for (auto e : c->timer.ev) cudaEventDestroy(e);
    comm_release(c);
    if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
    delete c;
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
        if ((rc0 = comm_init(c, dist))) return bail(rc0);
        c->use_graph = false;   // collectives stay outside graphs
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
    if (k == "graph") { c->use_graph = value != 0 && c->world == 1 && !c->loop_nccl; drop_graphs(); return GBS_OK; }
    if (k == "time_kernels") { c->time_kernels = value != 0; drop_graphs(); return GBS_OK; }
    if (k == "overlap") { c->use_overlap = value != 0; drop_graphs(); return GBS_OK; }
    if (k == "l2hint") { c->hint_opt = (int)std::max<int64_t>(0, value); drop_graphs(); return GBS_OK; }
    if (k == "l2hint_step") { c->hint_step_opt = (int)std::max<int64_t>(0, value); drop_graphs(); return GBS_OK; }
    if (k == "band") { c->band_opt = (int)std::max<int64_t>(0, value); drop_graphs(); return GBS_OK; }
    if (k == "fin_ring") { c->fin_ring = value != 0; drop_graphs(); return GBS_OK; }
    if (k == "fea_ring") { c->fea_ring = value != 0; drop_graphs(); return GBS_OK; }
    if (k == "fea") { c->use_fea = value != 0; drop_graphs(); return GBS_OK; }
    if (k == "streams") {
        if (value != 1 && value != 2) return fail(c, GBS_E_INVAL, "streams must be 1 or 2");
        c->n_streams = (int)value; drop_graphs(); return GBS_OK;
    }
    if (k == "zchunk_fin") { c->zchunk_fin_opt = (int)std::max<int64_t>(0, value); drop_graphs(); return GBS_OK; }
    if (k == "l2hint_fin") { c->hint_fin_opt = (int)std::max<int64_t>(0, value); drop_graphs(); return GBS_OK; }
    if (k == "zchunk_pair") { c->zchunk_pair_opt = (int)std::max<int64_t>(0, value); drop_graphs(); return GBS_OK; }
    if (k == "zchunk") { c->zchunk_opt = (int)std::max<int64_t>(0, value); drop_graphs(); return GBS_OK; }
    if (k == "bulk") { c->use_bulk = value != 0; drop_graphs(); return GBS_OK; }
    if (k == "fuse") { c->use_fuse = value != 0; drop_graphs(); return GBS_OK; }
    if (k == "fuse2d") { c->use_fuse2d = value != 0; drop_graphs(); return GBS_OK; }
    if (k == "half") { c->use_half = value != 0; drop_graphs(); return GBS_OK; }
    if (k == "half_fe") { c->half_fe = value != 0; drop_graphs(); return GBS_OK; }
    if (k == "half_tall") { c->half_tall = value != 0; drop_graphs(); return GBS_OK; }
    if (k == "half_rpt") {
        if (value != 2 && value != 4) return fail(c, GBS_E_INVAL, "half_rpt must be 2 or 4");
        c->half_rpt = (int)value; drop_graphs(); return GBS_OK;
    }
    if (k == "l2hint_half") { c->hint_half_opt = (int)std::max<int64_t>(0, value); drop_graphs(); return GBS_OK; }
    if (k == "loopback_nccl") {
        if (c->world > 1) return fail(c, GBS_E_UNSUPPORTED, "loopback_nccl needs a single-GPU context");
        const bool on = value != 0;
        if (on && !c->comm_slab) {
            int rc = comm_nccl_self(c, &c->comm_slab);
            if (rc) return rc;
        }
        cudaStreamSynchronize(c->stream);
        drop_graphs();
        c->loop_nccl = on;
        c->use_graph = !on && c->use_graph;   // NCCL calls stay outside graphs, as with world > 1
        return GBS_OK;
    }
    if (k == "peer") {
        // loopback slabs on one GPU: the peer-push path with the neighbouring slabs' buffers
        const bool on = value != 0;
        if (on && !peer_eligible(c, false))
            return fail(c, GBS_E_UNSUPPORTED, "peer pushes need loopback slabs of a 3-D TMA grid (fuse, bulk on)");
        cudaStreamSynchronize(c->stream);
        drop_graphs();
        if (on && !c->d_peer_flags) {
            CU(c, cudaMalloc(&c->d_peer_flags, sizeof(unsigned long long) * 2 * c->loopback));
            CU(c, cudaMemset(c->d_peer_flags, 0, sizeof(unsigned long long) * 2 * c->loopback));
            c->peer_epoch = 0;
        }
        c->peer_on = on;
        c->peer_ghosts_valid = false;
        return GBS_OK;
    }
    if (k == "persistent") { c->use_persistent = value != 0; return GBS_OK; }
    if (k == "fused_combine") {
        // the final pass stores into the owners' staging slots of the other group members'
        // contexts: needs groups > 1 with the members in this process (local transport)
        if (value && (c->groups < 2 || !c->comm_group || (!c->local_transport && c->grp_ws.empty())))
            return fail(c, GBS_E_UNSUPPORTED, "fused_combine needs sequence groups whose contexts share this "
                                              "process (GBS_TRANSPORT_LOCAL) or gbs_bind_group_peers");
        c->fused_combine = value != 0;
        drop_graphs();
        return GBS_OK;
    }
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
        if (c->d_peer_flags) { cudaFree(c->d_peer_flags); c->d_peer_flags = nullptr; }
        c->peer_on = false;
        return alloc_state(c);
    }
    return fail(c, GBS_E_INVAL, "unknown option '%s'", key);
}

int gbs_workspace_bytes(const gbs_ctx* c, int64_t* bytes) {
    if (!c || !bytes) return fail(const_cast<gbs_ctx*>(c), GBS_E_INVAL, "ctx or bytes is NULL");
    *bytes = state_bytes(c) + kPeerFlagBytes;     // + this rank's peer flags (gbs_bind_peers)
    return GBS_OK;
}

int gbs_bind_workspace(gbs_ctx* c, void* device_ptr, int64_t bytes) {
    if (!c) return fail(c, GBS_E_INVAL, "ctx is NULL");
    if (device_ptr && bytes < state_bytes(c) + kPeerFlagBytes)
        return fail(c, GBS_E_INVAL, "workspace of %lld bytes < %lld (gbs_workspace_bytes)", (long long)bytes,
                    (long long)(state_bytes(c) + kPeerFlagBytes));
    if (device_ptr && (reinterpret_cast<uintptr_t>(device_ptr) % 256))
        return fail(c, GBS_E_INVAL, "workspace must be 256-byte aligned");
    CU(c, cudaSetDevice(c->device));
    CU(c, cudaStreamSynchronize(c->stream));
    int rc = consume_in(c);
    if (rc) return rc;
    CU(c, cudaStreamSynchronize(c->stream));
    for (auto& g : c->gexec) if (g) { cudaGraphExecDestroy(g); g = nullptr; }
    free_state(c);                      // own buffers are released; a workspace is only forgotten
    c->ws_ptr = device_ptr;
    c->ws_bytes = device_ptr ? bytes : 0;
    c->have_state = false;              // the state must be written again
    c->peer_on = false;                 // peers are bound to a workspace
    c->peer_base[0] = c->peer_base[1] = nullptr;
    if (!c->grp_ws.empty()) c->fused_combine = false;   // so are the group members'
    c->grp_ws.clear();
    c->grp_stage.clear();
    if (device_ptr) {
        CU(c, cudaMemset(static_cast<char*>(device_ptr) + state_bytes(c), 0, kPeerFlagBytes));
        c->peer_flags_fresh = true;
    }
    return GBS_OK;
}

int gbs_bind_peers(gbs_ctx* c, void* lower_workspace, void* upper_workspace) {
    if (!c) return fail(c, GBS_E_INVAL, "ctx is NULL");
    if (!lower_workspace || !upper_workspace) {
        c->peer_on = false;
        c->peer_base[0] = c->peer_base[1] = nullptr;
        return GBS_OK;
    }
    if (!c->ws_ptr) return fail(c, GBS_E_STATE, "gbs_bind_peers needs a bound workspace (gbs_bind_workspace)");
    if (c->local_transport)
        return fail(c, GBS_E_UNSUPPORTED, "peer pushes between contexts of one process (local transport): their "
                                          "kernels would wait on one another's launches on one GPU");
    if (!peer_eligible(c, true))
        return fail(c, GBS_E_UNSUPPORTED, "peer pushes need pure z-slabs (groups = 1) of a 3-D TMA grid on >1 GPU");
    CU(c, cudaSetDevice(c->device));
    CU(c, cudaStreamSynchronize(c->stream));
    for (auto& g : c->gexec) if (g) { cudaGraphExecDestroy(g); g = nullptr; }
    c->peer_base[0] = static_cast<char*>(lower_workspace);
    c->peer_base[1] = static_cast<char*>(upper_workspace);
    // epochs restart only over freshly zeroed flags (gbs_bind_workspace, then a cross-rank
    // barrier by the caller before any rank binds); a re-bind keeps counting, so flags that
    // still hold earlier epochs never satisfy a wait early
    if (c->peer_flags_fresh) c->peer_epoch = 0;
    c->peer_flags_fresh = false;
    c->peer_on = true;
    c->peer_ghosts_valid = false;
    return GBS_OK;
}

int gbs_stage_bytes(const gbs_ctx* c, int64_t* bytes) {
    if (!c || !bytes) return fail(const_cast<gbs_ctx*>(c), GBS_E_INVAL, "ctx or bytes is NULL");
    *bytes = c->groups > 1 ? stage_bytes_of(c) : 0;
    return GBS_OK;
}

int gbs_bind_group_peers(gbs_ctx* c, void* const* member_workspaces, void* const* member_stages, int n) {
    if (!c) return fail(c, GBS_E_INVAL, "ctx is NULL");
    if (n == 0 || !member_workspaces || !member_stages) {
        c->grp_ws.clear();
        c->grp_stage.clear();
        c->fused_combine = false;
        return GBS_OK;
    }
    if (c->groups < 2 || n != c->groups)
        return fail(c, GBS_E_INVAL, "n=%d must equal the sequence groups (%d, >= 2)", n, c->groups);
    if (!c->ws_ptr) return fail(c, GBS_E_STATE, "gbs_bind_group_peers needs a bound workspace (gbs_bind_workspace)");
    if (member_workspaces[c->my_group] != c->ws_ptr)
        return fail(c, GBS_E_INVAL, "member_workspaces[my_group] is not this context's workspace");
    for (int j = 0; j < n; ++j)
        if (!member_workspaces[j] || !member_stages[j]) return fail(c, GBS_E_INVAL, "member %d pointer is NULL", j);
    CU(c, cudaSetDevice(c->device));
    CU(c, cudaStreamSynchronize(c->stream));
    c->grp_ws.assign(n, nullptr);
    c->grp_stage.assign(n, nullptr);
    for (int j = 0; j < n; ++j) {
        c->grp_ws[j] = static_cast<char*>(member_workspaces[j]);
        c->grp_stage[j] = static_cast<char*>(member_stages[j]);
    }
    c->fused_combine = true;
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
    if (!c || cls < 0 || cls > 7) return fail(c, GBS_E_INVAL, "ctx NULL or cls out of range");
    int rc = harvest_timer(c);
    if (rc) return rc;
    if (total_ms) *total_ms = c->timer.total_ms[cls];
    if (launches) *launches = c->timer.launches[cls];
    if (reset) { c->timer.total_ms[cls] = 0; c->timer.launches[cls] = 0; }
    return GBS_OK;
}

}  // extern "C"

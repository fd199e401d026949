// gbs_io.cu -- state IO: full-grid and slab-local reads and writes (host or
// device buffers), the asynchronous slab IO on the context's own copy streams,
// gbs_sync and the deferred non-finite check.
#include "gbs_internal.h"

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
            for (double* p : c->in_buf) cudaFree(p);          // all slabs or none
            for (double* p : c->out_buf) cudaFree(p);
            c->in_buf.clear();
            c->out_buf.clear();
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
void async_release(gbs_ctx* c) {
    if (c->h2d) cudaStreamSynchronize(c->h2d);
    if (c->d2h) cudaStreamSynchronize(c->d2h);
    for (double* p : c->in_buf) cudaFree(p);
    for (double* p : c->out_buf) cudaFree(p);
    c->in_buf.clear();
    c->out_buf.clear();
    c->pending_in = false;
}

// a staged incoming state becomes Y (in context-stream order)
int consume_in(gbs_ctx* c) {
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

int check_flag(gbs_ctx* c) {
    int h = 0;
    CU(c, cudaMemcpyAsync(&h, c->d_flag, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    CU(c, cudaStreamSynchronize(c->stream));
    if (h) {
        CU(c, cudaMemsetAsync(c->d_flag, 0, sizeof(int), c->stream));
        return fail(c, GBS_E_NONFINITE, "non-finite state after a macro step (H beyond the stability limit?)");
    }
    return GBS_OK;
}

// this rank's planes [z_lo, z_lo + nz_rank) of the slowest axis (all its local slabs)
static void rank_planes(const gbs_ctx* c, int64_t* z_lo, int64_t* nz_rank) {
    *z_lo = c->slab[0].z0;
    *nz_rank = 0;
    for (const auto& s : c->slab) *nz_rank += s.nz;
}

extern "C" {

int gbs_write_state(gbs_ctx* c, const double* src, int64_t count, int on_device) {
    if (!c || !src) return fail(c, GBS_E_INVAL, "ctx or src is NULL");
    if (count != c->F * c->points)
        return fail(c, GBS_E_INVAL, "count=%lld, expected F*points=%lld", (long long)count, (long long)(c->F * c->points));
    CU(c, cudaSetDevice(c->device));
    int rc0 = consume_in(c);
    if (!rc0) rc0 = ensure_buffers(c);
    if (rc0) return rc0;
    const cudaMemcpyKind kind = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    for (auto& s : c->slab)
        for (int f = 0; f < c->F; ++f)
            CU(c, cudaMemcpyAsync(field_ptr(c, s, c->yb, f), src + (int64_t)f * c->points + s.z0 * c->plane,
                                  sizeof(double) * (size_t)(s.nz * c->plane), kind, c->stream));
    c->have_state = true;
    c->peer_ghosts_valid = false;        // peer mode refills Y's ghost planes at the next advance
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

static int read_state_impl(gbs_ctx* c, double* dst, int64_t count, int on_device);

int gbs_read_state(gbs_ctx* c, double* dst, int64_t count, int on_device) {
    return comm_abort_on_error(c, read_state_impl(c, dst, count, on_device));
}

}  // extern "C"

static int read_state_impl(gbs_ctx* c, double* dst, int64_t count, int on_device) {
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
        Slab& s = c->slab[0];
        const size_t slab_cnt = (size_t)(s.nz * c->plane);
        if (!c->d_gather) CU(c, cudaMalloc(&c->d_gather, sizeof(double) * (size_t)c->points));
        for (int f = 0; f < c->F; ++f) {
            int rc = c->comm_slab->allgather(c, field_ptr(c, s, c->yb, f), c->d_gather, slab_cnt, c->stream);
            if (rc) return rc;
            CU(c, cudaMemcpyAsync(dst + (int64_t)f * c->points, c->d_gather, sizeof(double) * (size_t)c->points,
                                  kind, c->stream));
        }
    }
    int rc = gbs_sync(c);
    if (rc) return rc;
    return harvest_timer(c);
}

extern "C" {

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
    if (!rc0) rc0 = ensure_buffers(c);
    if (rc0) return rc0;
    const cudaMemcpyKind kind = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    for (auto& s : c->slab)
        for (int f = 0; f < c->F; ++f)
            CU(c, cudaMemcpyAsync(field_ptr(c, s, c->yb, f), src + (int64_t)f * per_field + (s.z0 - z_lo) * c->plane,
                                  sizeof(double) * (size_t)(s.nz * c->plane), kind, c->stream));
    c->have_state = true;
    c->peer_ghosts_valid = false;        // peer mode refills Y's ghost planes at the next advance
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
    if ((rc = ensure_buffers(c))) return rc;
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
    c->peer_ghosts_valid = false;        // peer mode refills Y's ghost planes at the next advance
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

}  // extern "C"

// gbs_plan.cu -- validation of a context's arguments, the planner (sequence
// groups balanced by sum(n_k + 1) x slabs of the slowest axis, SURVEY.md §8(e),
// PAPER.md:388-400) and the per-slab halo schedule; the host-only ABI queries
// gbs_plan / gbs_halo_schedule expose exactly what gbs_create uses.
#include "gbs_internal.h"

// ---------------------------------------------------------------------------
// planning
// ---------------------------------------------------------------------------
// Partition sequence indices into g groups minimising the largest group load
// sum(n_k + 1) (§3.6: sequences folded onto cores so that
// every core does the same number of RHS evaluations; exact
// search, m <= 32).  Exact branch and bound: sequences in descending load,
// each placed into a group whose load stays below the best maximum found so
// far, never into two groups of equal load (symmetry), stopped at the lower
// bound max(ceil(total / g), largest load).  The initial bound is the LPT
// (longest processing time first) partition, which is also the answer if the
// search exceeds its node budget (never for the step sets of the configs and
// the paper's schemes, which finish in well under a millisecond).
namespace {
struct PartitionSearch {
    std::vector<int64_t> w;           // loads, descending
    int g = 1;
    int64_t lower = 0, best = 0;
    std::vector<int> cur, best_asg;   // group of each item
    std::vector<int64_t> load;
    int64_t nodes = 0, budget = 20000000;
    void dfs(size_t i, int64_t cur_max) {
        if (best == lower || nodes > budget) return;
        ++nodes;
        if (i == w.size()) {
            if (cur_max < best) { best = cur_max; best_asg = cur; }
            return;
        }
        for (int q = 0; q < g; ++q) {
            bool dup = false;             // a group with the same load was tried already
            for (int p = 0; p < q; ++p)
                if (load[p] == load[q]) { dup = true; break; }
            if (dup) continue;
            const int64_t nl = load[q] + w[i];
            if (nl >= best) continue;
            load[q] = nl;
            cur[i] = q;
            dfs(i + 1, std::max(cur_max, nl));
            load[q] -= w[i];
            if (best == lower || nodes > budget) return;
        }
    }
};
}  // namespace

std::vector<std::vector<int>> partition(const std::vector<int>& nk, int g) {
    const int m = (int)nk.size();
    std::vector<int> order(m);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return nk[a] > nk[b]; });
    PartitionSearch P;
    P.g = std::max(1, g);
    int64_t total = 0;
    for (int i : order) { P.w.push_back(nk[i] + 1); total += nk[i] + 1; }
    P.lower = m ? std::max<int64_t>((total + P.g - 1) / P.g, P.w[0]) : 0;
    // LPT: the starting bound and the fallback
    std::vector<int64_t> load(P.g, 0);
    P.best_asg.assign(m, 0);
    for (int j = 0; j < m; ++j) {
        int q = (int)(std::min_element(load.begin(), load.end()) - load.begin());
        P.best_asg[j] = q;
        load[q] += P.w[j];
    }
    P.best = m ? *std::max_element(load.begin(), load.end()) : 0;
    if (P.best > P.lower) {
        P.cur.assign(m, 0);
        P.load.assign(P.g, 0);
        P.dfs(0, 0);
    }
    std::vector<std::vector<int>> grp(P.g);
    for (int j = 0; j < m; ++j) grp[P.best_asg[j]].push_back(order[j]);
    // deterministic group order: descending largest step count (empty groups last)
    std::stable_sort(grp.begin(), grp.end(), [&](const std::vector<int>& a, const std::vector<int>& b) {
        const int ma = a.empty() ? -1 : nk[a[0]], mb = b.empty() ? -1 : nk[b[0]];
        return ma > mb;
    });
    for (auto& v : grp) std::sort(v.begin(), v.end(), [&](int a, int b) { return nk[a] < nk[b]; });
    return grp;
}

int64_t crit_path(const std::vector<int>& nk, int g) {
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
void plan(gbs_ctx* c, int want_groups) {
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
// The per-substep halo schedule of one slab (posted inside one NCCL group).
// Per field: send up (my top interior planes -> the upper neighbour's low
// ghosts), send down (my bottom interior planes -> the lower neighbour's high
// ghosts), receive from below (into my low ghosts), receive from above (into
// my high ghosts).  NCCL matches p2p operations per peer pair in posting order:
// slab a's k-th send to b is b's k-th receive from a.  With 2 slabs both
// neighbours are the same peer and the order send-up/send-down vs
// recv-low/recv-high pairs a's top planes with b's low ghosts -- as required.
// ---------------------------------------------------------------------------
std::vector<gbs_halo_op> halo_schedule(int slabs, int my_slab, int64_t nz, int G, unsigned mask) {
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

// Validate the grid and the scheme (weights only when w_k != NULL) into c.
int validate(gbs_ctx* c, const gbs_grid* g, int stencil_order, int m, const int32_t* n_k,
                    const double* w_k) {
    c->pde = g->pde;
    if (g->pde == GBS_ADV1D) { c->ndim = 1; c->F = 1; }
    else if (g->pde == GBS_ACOUSTIC2D) { c->ndim = 2; c->F = 3; }
    else if (g->pde == GBS_WAVE3D) { c->ndim = 3; c->F = 2; }
    else return fail(c, GBS_E_INVAL, "grid.pde=%d is not a known PDE", g->pde);
    if (g->ndim != c->ndim) return fail(c, GBS_E_INVAL, "grid.ndim=%d does not match the PDE", g->ndim);
    if (stencil_order == 0) {
        // spectral derivative: 1-D advection on an even grid -- the whole run
        // in the cluster kernel (N <= kSpectralMaxN, m <= 16, one GPU), else cuFFT per substep
        if (g->pde != GBS_ADV1D)
            return fail(c, GBS_E_INVAL, "stencil_order=0 (spectral) is defined for GBS_ADV1D only");
        if (g->n[0] < 4 || g->n[0] % 2 || g->n[0] > (1LL << 30))
            return fail(c, GBS_E_INVAL, "spectral grid n[0]=%lld must be even, 4..2^30", (long long)g->n[0]);
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
int make_plan(gbs_ctx* c, int rank, int world, int groups) {
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

extern "C" {

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

}  // extern "C"

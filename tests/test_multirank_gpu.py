"""The multi-GPU path, executed: N ranks as N contexts of one process on one B200, joined
by the in-process transport (GBS_TRANSPORT_LOCAL, include/gbs.h) and driven by N host
threads.  Everything a rank does on N GPUs runs: gbs_create's communicator split, the
sequence-group x slab plan, the per-group FE / LF / FIN0-FINACC chains, the per-substep
halo schedule (matched in NCCL's posting order), the combine across sequence groups
(PAPER.md:109-115 -- "the approximations ... are combined"; §3.6 folding, 388-400) and the
slab all-gather of gbs_read_state.  Only the transport differs (device copies ordered by
events instead of NCCL over NVLink; no kernel waits on another rank's kernel).

Bar: every rank's full state within 1e-12 relative L2 of the oracle (per field and over all
fields) and max |error| per element within 1e-11 of max |state|; pure slabs (groups = 1) are
bit-identical to the one-context run (same arithmetic per point; halos are exact copies).
"""

import numpy as np
import pytest

from gbs_inputs import get_config, make_ic, reduced
from oracle import c_oracle as C
from oracle import stability as S
from oracle import weights as W

from conftest import record_parity

pytestmark = pytest.mark.gpu
TOL = 1e-12
TOL_ELEM = 1e-11      # per element, relative to max |ref|


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1907_11771_b200 import gbs
    gbs.load()
    return torch


def scheme_for(w, wset, cfg):
    counts, ws, _ = W.scheme(wset, w.steps)
    wd = W.to_double(ws)
    H = S.macro_step_H(w.pde, w.order, w.n, counts, wd, w.h_factor)
    # parity-only sets use min(H_config, 0.5 ISB(set)/rho) (reading R7)
    cf, wf, _ = W.scheme(get_config(cfg).weights, w.steps)
    H = min(H, S.macro_step_H(w.pde, w.order, w.n, cf, W.to_double(wf), w.h_factor))
    return counts, wd, H


def errors(got, ref):
    """(max relative L2 over fields and all fields, max |err| / RMS(ref), max |err| / max |ref|)."""
    rel = [float(np.linalg.norm((got[f] - ref[f]).ravel()) / np.linalg.norm(ref[f].ravel()))
           for f in range(ref.shape[0]) if np.linalg.norm(ref[f]) > 0]
    rel.append(float(np.linalg.norm((got - ref).ravel()) / np.linalg.norm(ref.ravel())))
    rms = float(np.sqrt(np.mean(ref.astype(np.float64) ** 2)))
    emax = float(np.max(np.abs(got - ref)))
    return max(rel), emax / rms, emax / float(np.max(np.abs(ref)))


def run_ranks(torch, w, counts, wd, H, M, world, groups, opts=None):
    from paper_1907_11771_b200 import gbs
    y0 = make_ic(w)

    def body(dist):
        torch.cuda.set_device(0)
        s = torch.cuda.Stream()
        with gbs.Stepper(w.pde, w.n, w.order, counts, wd, dist=dist, stream=s.cuda_stream,
                         **(opts or {})) as st:
            st.write(y0)
            st.advance(M, H)
            out = np.empty_like(y0)
            st.read(out)
            return out, st.info()

    res = gbs.run_local_ranks(world, body, groups=groups)
    return y0, [r[0] for r in res], [r[1] for r in res]


def run_single(torch, w, counts, wd, H, M, opts=None):
    from paper_1907_11771_b200 import gbs
    y0 = make_ic(w)
    with gbs.Stepper(w.pde, w.n, w.order, counts, wd, **(opts or {})) as st:
        st.write(y0)
        st.advance(M, H)
        out = np.empty_like(y0)
        st.read(out)
    return out


def check(torch, cfg, n, M, world, groups, wset="nonzero8", opts=None):
    w = reduced(cfg, n, macro_steps=M, weights=wset)
    counts, wd, H = scheme_for(w, wset, cfg)
    y0, outs, infos = run_ranks(torch, w, counts, wd, H, M, world, groups, opts)
    # the plan that ran: g groups x s slabs, every sequence in exactly one group
    g = infos[0]["groups"]
    assert g == groups and infos[0]["slabs"] == world // groups
    seqs = {}
    for r, info in enumerate(infos):
        assert info["my_group"] * (world // groups) + info["my_slab"] == r
        seqs[info["my_group"]] = info["my_substeps"]
    assert sum(seqs.values()) == sum(k + 1 for k in counts)
    # every rank gathered the same full state
    for o in outs[1:]:
        assert np.array_equal(o, outs[0])
    ref = C.advance(w.pde, w.order, y0, counts, wd, H, M)
    rel, mrms, mmax = errors(outs[0], ref)
    record_parity(f"multirank {cfg} {n} {wset} world={world} groups={groups} {opts or {}}", rel, mrms, mmax)
    assert rel <= TOL and mmax <= TOL_ELEM, f"{cfg} {n} world={world} groups={groups}: rel L2 {rel:.3e}, max {mmax:.3e}"
    single = run_single(torch, w, counts, wd, H, M, {k: v for k, v in (opts or {}).items() if k != "fused_combine"})
    if groups == 1:
        assert np.array_equal(outs[0], single), "pure slabs must be bit-identical to one context"
    else:
        rel1, _, mmax1 = errors(outs[0], single)
        assert rel1 <= TOL and mmax1 <= TOL_ELEM
    return rel, mmax


# 3-D wave, C4 scheme ({2..12}), two-substep TMA path (grid of whole 64 x 16 tiles)
@pytest.mark.parametrize("world,groups", [(2, 1), (2, 2), (4, 1), (4, 2), (4, 4), (8, 1), (8, 2), (8, 4)])
def test_wave3d_c4_scheme_tma(torch_cuda, world, groups):
    check(torch_cuda, "c4", (64, 32, 48), 2, world, groups)


# 3-D wave, C4 scheme, ragged grid (register kernels, odd x tail)
@pytest.mark.parametrize("world,groups", [(2, 1), (2, 2), (4, 2), (8, 2)])
def test_wave3d_c4_scheme_ragged(torch_cuda, world, groups):
    check(torch_cuda, "c4", (70, 34, 48), 2, world, groups)


# 3-D wave, C5 scheme ({2..16}), TMA path; slabs thick enough for the overlapped exchange
@pytest.mark.parametrize("world,groups", [(2, 1), (4, 2), (4, 4), (8, 1), (8, 2), (8, 4)])
def test_wave3d_c5_scheme_tma(torch_cuda, world, groups):
    check(torch_cuda, "c5", (128, 16, 96), 2, world, groups)


def test_wave3d_c5_scheme_fallback_weights(torch_cuda):
    """The bench's weight set (zero weights on 10..16, sequences still run)."""
    check(torch_cuda, "c5", (64, 16, 64), 2, 4, 2, wset="fallback8")


# 2-D acoustics (slabs along y; p and v cross them): C2 (FD4) and C3 (FD8) schemes
@pytest.mark.parametrize("cfg,n,world,groups", [("c3", (128, 64, 1), 2, 1), ("c3", (128, 64, 1), 2, 2),
                                                ("c3", (128, 64, 1), 4, 2), ("c2", (96, 80, 1), 4, 1),
                                                ("c2", (64, 128, 1), 8, 2), ("c3", (128, 96, 1), 4, 4)])
def test_acoustic2d(torch_cuda, cfg, n, world, groups):
    check(torch_cuda, cfg, n, 2, world, groups)


# 1-D advection: sequence groups only (1-D grids are not slabbed)
@pytest.mark.parametrize("world", [2, 4])
def test_adv1d_groups(torch_cuda, world):
    check(torch_cuda, "c1", (256, 1, 1), 5, world, world, wset="square8")


@pytest.mark.parametrize("opts", [{"overlap": 0}, {"fuse": 0}, {"bulk": 0}])
def test_wave3d_options_across_ranks(torch_cuda, opts):
    """The exchange-then-compute path, single-substep kernels and register kernels across ranks."""
    check(torch_cuda, "c4", (64, 32, 64), 2, 4, 2, opts=opts)


def test_planner_choice_runs(torch_cuda):
    """groups = 0: the planner's own choice for 8 ranks executes and matches the oracle."""
    from paper_1907_11771_b200 import gbs
    w = reduced("c5", (128, 16, 64), macro_steps=1, weights="nonzero8")
    counts, wd, H = scheme_for(w, "nonzero8", "c5")
    plan = gbs.gbs_plan(w.pde, w.n, w.order, counts, 8, 0, 0)
    check(torch_cuda, "c5", (128, 16, 64), 1, 8, plan["groups"])


# fused combine: the final pass stores into the owners' staging slots, owners sum
# their plane range in member order and store into every member -- bit-identical to the
# transport's all-reduce (same sums, same order) and the oracle's result within the bar
@pytest.mark.parametrize("cfg,n,world,groups", [("c4", (64, 32, 48), 2, 2), ("c4", (64, 32, 48), 4, 2),
                                                ("c5", (128, 16, 96), 8, 4), ("c5", (64, 16, 64), 4, 4),
                                                ("c5", (64, 16, 64), 8, 8)])
def test_fused_combine_equals_allreduce(torch_cuda, cfg, n, world, groups):
    w = reduced(cfg, n, macro_steps=2, weights="nonzero8")
    counts, wd, H = scheme_for(w, "nonzero8", cfg)
    y0, a, ia = run_ranks(torch_cuda, w, counts, wd, H, 2, world, groups, {"fused_combine": 1})
    _, b, ib = run_ranks(torch_cuda, w, counts, wd, H, 2, world, groups, {"fused_combine": 0})
    for r in range(world):
        assert np.array_equal(a[r], b[r])
    ref = C.advance(w.pde, w.order, y0, counts, wd, H, 2)
    rel, mrms, mmax = errors(a[0], ref)
    record_parity(f"multirank fused combine {cfg} {n} world={world} groups={groups}", rel, mrms, mmax)
    assert rel <= TOL and mmax <= TOL_ELEM


def test_fused_combine_rejected_without_local_groups(torch_cuda):
    from paper_1907_11771_b200 import gbs
    w = reduced("c4", (64, 32, 24), macro_steps=1, weights="nonzero8")
    counts, wd, _ = scheme_for(w, "nonzero8", "c4")
    with gbs.Stepper(w.pde, w.n, w.order, counts, wd) as st:       # one context, no groups
        with pytest.raises(gbs.GbsError) as e:
            gbs.gbs_set_option(st.ctx, "fused_combine", 1)
        assert e.value.code == gbs.GBS_E_UNSUPPORTED


@pytest.mark.parametrize("world,groups", [(2, 2), (4, 2), (8, 4)])
def test_fused_combine_through_bound_peer_buffers(torch_cuda, world, groups):
    """The multi-GPU form of the fused combine: each rank binds a torch workspace and a staging
    tensor, and every group member's pair of addresses (peer memory across GPUs; the same device
    here) through gbs_bind_group_peers.  Bit-identical to the all-reduce."""
    import threading
    from paper_1907_11771_b200 import gbs
    w = reduced("c5", (64, 16, 64), macro_steps=2, weights="nonzero8")
    counts, wd, H = scheme_for(w, "nonzero8", "c5")
    y0 = make_ic(w)
    slabs = world // groups
    ptrs = [None] * world
    bar = threading.Barrier(world)

    def body(dist):
        torch = torch_cuda
        torch.cuda.set_device(0)
        s = torch.cuda.Stream()
        r = dist["rank"]
        with gbs.Stepper(w.pde, w.n, w.order, counts, wd, dist=dist, stream=s.cuda_stream,
                         torch_memory=True) as st:
            stage = torch.empty(max(gbs.gbs_stage_bytes(st.ctx), 1), dtype=torch.uint8, device="cuda")
            ptrs[r] = (st.workspace.data_ptr(), stage.data_ptr())
            bar.wait()
            me = st.info()
            members = [j * slabs + me["my_slab"] for j in range(groups)]
            gbs.gbs_bind_group_peers(st.ctx, [ptrs[m][0] for m in members], [ptrs[m][1] for m in members])
            st.write(y0)
            st.advance(2, H)
            out = np.empty_like(y0)
            st.read(out)
            bar.wait()                     # every member done before any staging tensor is freed
            return out

    a = gbs.run_local_ranks(world, body, groups=groups)
    _, b, _ = run_ranks(torch_cuda, w, counts, wd, H, 2, world, groups, {"fused_combine": 0})
    for r in range(world):
        assert np.array_equal(a[r], b[r])


@pytest.mark.slow
@pytest.mark.parametrize("world,groups,fused", [(8, 2, 1), (8, 1, 0), (4, 4, 1)])
def test_c4_full_size_multirank(torch_cuda, world, groups, fused):
    """The C4 grid at full size (512^3, FD8, {2..12}, nonzero8) as 4-8 ranks (slabs of 64-512
    planes, sequence groups, the fused combine) on one GPU, one macro step, full state."""
    opts = {"fused_combine": fused} if groups > 1 else {}
    rel, mmax = check(torch_cuda, "c4", (512, 512, 512), 1, world, groups, opts=opts)
    assert rel <= TOL


@pytest.mark.slow
@pytest.mark.parametrize("groups,fused", [(1, 0)])
def test_c5_full_size_eight_ranks_match_one_context(torch_cuda, groups, fused):
    """The bench workload itself (C5: 1024^3, FD8, {2..16}, fallback8) as 8 ranks on one GPU --
    the decomposition the 8-GPU bench runs (the planner's pure slabs of 128 planes) -- one macro
    step, every rank's slab bit-identical to the one-context state.  (Sequence groups at this
    size do not fit one GPU's memory: 8 ranks x 6 buffers x 4 GiB; C4 covers them at full size.)"""
    from paper_1907_11771_b200 import gbs
    torch = torch_cuda
    w = get_config("c5")
    counts, wd, H = scheme_for(w, "fallback8", "c5")
    y0 = make_ic(w)
    with gbs.Stepper(w.pde, w.n, w.order, counts, wd) as st:
        st.write(torch.from_numpy(y0).cuda())
        st.advance(1, H)
        ref = np.empty_like(y0)
        st.read(ref)
    world = 8

    def body(dist):
        torch.cuda.set_device(0)
        s = torch.cuda.Stream()
        opts = {"fused_combine": fused} if groups > 1 else {}
        with gbs.Stepper(w.pde, w.n, w.order, counts, wd, dist=dist, stream=s.cuda_stream, **opts) as st:
            info = st.info()
            z0, nz = info["slab_z0"], info["slab_nz"]
            st.write_slab(np.ascontiguousarray(y0[:, z0:z0 + nz]))
            st.advance(1, H)
            out = np.empty((2, nz) + y0.shape[2:], dtype=np.float64)
            st.read_slab(out)
            return z0, nz, out, info["groups"]

    res = gbs.run_local_ranks(world, body, groups=groups)
    for z0, nz, out, g in res:
        assert g == groups
        part = ref[:, z0:z0 + nz]
        if groups == 1:
            assert np.array_equal(out, part)
        else:
            rel, _, mmax = errors(out, part)
            assert rel <= TOL and mmax <= TOL_ELEM


def test_failed_rank_releases_the_others(torch_cuda):
    """A rank whose gbs_advance fails (here: an invalid H) marks its local communicators broken,
    so the other ranks blocked in a collective fail at once instead of after the 300 s timeout."""
    import time
    from paper_1907_11771_b200 import gbs
    w = reduced("c4", (64, 32, 48), macro_steps=1, weights="nonzero8")
    counts, wd, H = scheme_for(w, "nonzero8", "c4")
    y0 = make_ic(w)
    codes = [None, None]

    def body(dist):
        torch_cuda.cuda.set_device(0)
        s = torch_cuda.cuda.Stream()
        with gbs.Stepper(w.pde, w.n, w.order, counts, wd, dist=dist, stream=s.cuda_stream) as st:
            st.write(y0)
            try:
                st.advance(2, H if dist["rank"] == 0 else -1.0)
                st.sync()
                out = np.empty_like(y0)
                st.read(out)
            except gbs.GbsError as e:
                codes[dist["rank"]] = e.code
        return True

    t0 = time.time()
    gbs.run_local_ranks(2, body, groups=1)
    assert time.time() - t0 < 120
    assert codes[1] == gbs.GBS_E_INVAL and codes[0] == gbs.GBS_E_NCCL

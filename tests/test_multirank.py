"""The N > 1 path's host logic, on CPU with the gloo backend (world sizes 2 and 4).

* the plan (gbs_plan, the planner gbs_create uses) is consistent across ranks:
  sequence groups partition the step counts, slabs tile the slowest axis;
* the halo schedule (gbs_halo_schedule, the ops gbs_advance posts to NCCL) executed
  with gloo point-to-point fills every ghost plane with the right neighbour's planes,
  including 2 slabs where both neighbours are the same peer;
* the sequence-group decomposition (partial sums sum_{k in group} w_k y*_k combined
  by an all-reduce) reproduces the single-process oracle;
* the bench.py coordination helpers (id broadcast, barrier, max over ranks).
No GPU is used: compute is the oracle's, communication is gloo, the plan and the
schedule come from the C ABI (host-only entry points).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from gbs_inputs import make_ic, reduced
from paper_1907_11771_b200 import gbs


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(world, fn, *args):
    port = _free_port()
    mp.spawn(_entry, args=(world, port, fn, args), nprocs=world, join=True)


def _entry(rank, world, port, fn, args):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        fn(rank, world, *args)
    finally:
        dist.destroy_process_group()


# --------------------------------------------------------------------------- plan (single process)
@pytest.mark.parametrize("pde,n,order,steps", [
    ("wave3d", (1024, 1024, 1024), 8, (2, 4, 6, 8, 10, 12, 14, 16)),
    ("wave3d", (512, 512, 512), 8, (2, 4, 6, 8, 10, 12)),
    ("acoustic2d", (4096, 4096, 1), 8, (2, 4, 6, 8, 10, 12)),
    ("wave3d", (64, 64, 64), 8, tuple(range(2, 31, 2))),
])
@pytest.mark.parametrize("world", [1, 2, 4, 8])
@pytest.mark.parametrize("groups", [0, 1, 2])
def test_plan_is_a_partition(pde, n, order, steps, world, groups):
    if groups and world % groups:
        pytest.skip("groups must divide world")
    plans = [gbs.gbs_plan(pde, n, order, steps, world, r, groups) for r in range(world)]
    g, s = plans[0]["groups"], plans[0]["slabs"]
    assert g * s == world and all(p["groups"] == g and p["slabs"] == s for p in plans)
    if groups:
        assert g == groups
    nslow = n[{"wave3d": 2, "acoustic2d": 1}[pde]]
    by_group = {}
    for r, p in enumerate(plans):
        assert r == p["my_group"] * s + p["my_slab"]
        by_group.setdefault(p["my_group"], p["my_n_k"])
        assert by_group[p["my_group"]] == p["my_n_k"]          # same group -> same sequences
        assert p["slab_nz"] * s == nslow and p["slab_z0"] == p["my_slab"] * p["slab_nz"]
    allk = sorted(k for v in by_group.values() for k in v)
    assert allk == sorted(steps)                                # each sequence exactly once
    loads = [sum(k + 1 for k in v) for v in by_group.values()]
    assert max(loads) == plans[0]["critical_substeps"]


def test_plan_balances_like_the_paper():
    """§3.6: {2..10} on 3 cores folds to {10},{8,2},{6,4} (11 RHS each)."""
    plans = [gbs.gbs_plan("wave3d", (64, 64, 64), 8, [2, 4, 6, 8, 10], 3, r, 3) for r in range(3)]
    groups = sorted(sorted(p["my_n_k"]) for p in plans)
    assert groups == [[2, 8], [4, 6], [10]]
    # the paper shares the first evaluation within a core (11 RHS); the GPU path
    # recomputes it per sequence, so a folded pair costs 12
    assert plans[0]["critical_substeps"] == 12


@pytest.mark.parametrize("cores,nmax", [(6, 22), (8, 30)])
def test_plan_folds_the_papers_multicore_schemes(cores, nmax):
    """§3.6: with N_max = 4 n_cores - 2, the counts {2..N_max} fold onto
    n_cores cores as {N_max} and pairs summing to N_max -- GBS_8,6 on 6 GPUs, GBS_8,8 on 8
    (SURVEY.md §8(f) NEXT-1).  Without the shared first evaluation a pair costs N_max + 2."""
    assert nmax == 4 * cores - 2
    counts = list(range(2, nmax + 1, 2))
    plans = [gbs.gbs_plan("wave3d", (64, 64, 64), 8, counts, cores, r, cores) for r in range(cores)]
    groups = sorted(sorted(p["my_n_k"]) for p in plans)
    assert [nmax] in groups
    pairs = [g for g in groups if g != [nmax]]
    assert len(pairs) == cores - 1 and all(len(g) == 2 and sum(g) == nmax for g in pairs)
    assert sorted(n for g in groups for n in g) == counts
    assert plans[0]["critical_substeps"] == nmax + 2


# --------------------------------------------------------------------------- gloo, multi-process
def _halo_worker(rank, world, nz_local, ghost, nfields):
    """Each rank = one slab of a periodic z axis; global plane index in every value."""
    P = 6                                       # values per plane (tiny)
    nz = nz_local * world
    buf = np.full((nfields, nz_local + 2 * ghost, P), np.nan)
    z0 = rank * nz_local
    for f in range(nfields):
        for zl in range(nz_local):
            buf[f, ghost + zl, :] = 1000 * f + (z0 + zl) + 0.01 * np.arange(P)
    mask = (1 << nfields) - 1
    ops = gbs.gbs_halo_schedule(world, rank, nz_local, ghost, mask)
    t = torch.from_numpy(buf)
    reqs = []
    for op in ops:                               # posted in schedule order, like the NCCL group
        view = t[op["field"], ghost + op["plane0"]: ghost + op["plane0"] + op["planes"]]
        if op["kind"] == "send":
            reqs.append(dist.isend(view.contiguous(), op["peer"]))
        else:
            tmp = torch.empty_like(view)
            reqs.append((dist.irecv(tmp, op["peer"]), view, tmp))
    for r in reqs:
        if isinstance(r, tuple):
            r[0].wait()
            r[1].copy_(r[2])
        else:
            r.wait()
    for f in range(nfields):
        for g in range(1, ghost + 1):
            lo = (z0 - g) % nz
            hi = (z0 + nz_local - 1 + g) % nz
            assert np.allclose(buf[f, ghost - g], 1000 * f + lo + 0.01 * np.arange(P)), (rank, f, g)
            assert np.allclose(buf[f, ghost + nz_local - 1 + g], 1000 * f + hi + 0.01 * np.arange(P))
    assert not np.isnan(buf).any()


@pytest.mark.parametrize("world,nz_local,ghost,nfields", [(2, 8, 4, 1), (2, 6, 4, 3), (4, 5, 4, 2),
                                                          (3, 4, 2, 1), (4, 4, 4, 2)])
def test_halo_schedule_with_gloo(world, nz_local, ghost, nfields):
    _run(world, _halo_worker, nz_local, ghost, nfields)


def _group_sum_worker(rank, world, cfg, n, groups):
    from oracle import c_oracle, stability, weights
    w = reduced(cfg, n, macro_steps=1, weights="nonzero8")
    counts, ws, _ = weights.scheme(w.weights, w.steps)
    wd = weights.to_double(ws)
    H = stability.macro_step_H(w.pde, w.order, w.n, counts, wd)
    y0 = make_ic(w)
    plan = gbs.gbs_plan(w.pde, w.n, w.order, counts, world, rank, groups)
    assert plan["groups"] == groups
    mine = plan["my_n_k"]
    wmap = dict(zip(counts, wd))
    if plan["my_slab"] == 0:                      # one contribution per group
        part = c_oracle.advance(w.pde, w.order, y0, mine, [wmap[k] for k in mine], H, 1)
    else:
        part = np.zeros_like(y0)
    t = torch.from_numpy(part)
    dist.all_reduce(t)                            # the combine step (ncclAllReduce on GPUs)
    ref = c_oracle.advance(w.pde, w.order, y0, counts, wd, H, 1)
    err = np.linalg.norm(t.numpy() - ref) / np.linalg.norm(ref)
    assert err < 1e-13, err


@pytest.mark.parametrize("world,groups,cfg,n", [(2, 2, "c4", (24, 20, 16)), (4, 4, "c5", (20, 16, 24)),
                                                (4, 2, "c2", (48, 40, 1))])
def test_sequence_group_decomposition_with_gloo(world, groups, cfg, n):
    _run(world, _group_sum_worker, cfg, n, groups)


def _helpers_worker(rank, world):
    from paper_1907_11771_b200 import dist as pdist
    assert pdist.env() == (rank, world, rank) and pdist.active()
    payload = bytes(range(128)) if rank == 0 else None
    assert pdist.broadcast_bytes(payload, 0) == bytes(range(128))
    pdist.barrier(sync_cuda=False)
    assert pdist.max_over_ranks(10.0 + rank) == 10.0 + world - 1
    assert pdist.sum_over_ranks(1.0) == world
    got = pdist.gather_objects({"rank": rank})
    assert [g["rank"] for g in got] == list(range(world))
    recs = pdist.gather_objects({"sm_mhz": 1500.0 + rank, "sm_max_mhz": 1965.0,
                                 "reasons": ["sw_power_cap"] if rank == 1 else [], "samples": 2})
    m = pdist.merge_clocks(recs)
    assert m["sm_mhz"] == 1500.0 and m["reasons"] == ["sw_power_cap"] and m["samples"] == 2 * world
    assert len(m["per_rank"]) == world


@pytest.mark.parametrize("world", [2, 4])
def test_bench_coordination_helpers_with_gloo(world):
    _run(world, _helpers_worker)

"""GPU parity: the CUDA path (through the C ABI) against the oracle, element by element,
on the same seeded inputs.  Bar: max relative L2 <= 1e-12 in fp64 (BASELINE.json
north_star), per field and over all fields.  Weights and H are the oracle's.
"""

import os

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


def gbs_mod():
    from paper_1907_11771_b200 import gbs
    return gbs


def rel_l2(a, b):
    d = np.linalg.norm((a - b).ravel())
    n = np.linalg.norm(b.ravel())
    return float(d / n) if n > 0 else float(d)


def assert_parity(got, ref, tol=TOL, what=""):
    """max relative L2 (per field and over all fields) <= tol (north_star's bar), and per
    element max |got - ref| <= TOL_ELEM * max |ref| (a single wrong point cannot
    hide in the L2 norm of a large grid; rounding reaches ~1e-12 of the maximum, a wrong
    coefficient, halo plane or dropped term >= 1e-6)."""
    errs = [rel_l2(got[f], ref[f]) for f in range(ref.shape[0]) if np.linalg.norm(ref[f]) > 0]
    errs.append(rel_l2(got, ref))
    amax = float(np.max(np.abs(ref)))
    emax = float(np.max(np.abs(got - ref)))
    rms = float(np.sqrt(np.mean(np.square(ref))))
    record_parity(what, max(errs), emax / rms if rms > 0 else emax, emax / amax if amax > 0 else emax)
    assert max(errs) <= tol, f"{what}: rel L2 per field/all = {errs}"
    assert emax <= TOL_ELEM * max(amax, 1e-300), f"{what}: max |err| / max |ref| = {emax / amax:.3e}"
    for f in range(ref.shape[0]):
        if np.linalg.norm(ref[f]) == 0:
            assert np.max(np.abs(got[f])) <= tol * max(1.0, np.linalg.norm(ref) / np.sqrt(ref.size))


def scheme_for(w, wset=None):
    counts, ws, _ = W.scheme(wset or w.weights, w.steps)
    wd = W.to_double(ws)
    H = S.macro_step_H(w.pde, w.order, w.n, counts, wd, w.h_factor)
    if wset and wset != w.weights:
        # parity-only sets use min(H_config, 0.5 ISB(set)/rho) (reading R7)
        c0, w0, _ = W.scheme(w.weights, w.steps)
        H = min(H, S.macro_step_H(w.pde, w.order, w.n, c0, W.to_double(w0), w.h_factor))
    return counts, wd, H


def run_gpu(torch, w, counts, wd, H, M, checkpoints=False, opts=None, host=False):
    gbs = gbs_mod()
    y0 = make_ic(w)
    outs = []
    with gbs.Stepper(w.pde, w.n, w.order, counts, wd, **(opts or {})) as st:
        if host:
            st.write(y0)
        else:
            st.write(torch.from_numpy(y0).cuda())
        steps = [1] * M if checkpoints else [M]
        for k in steps:
            st.advance(k, H)
            if host:
                o = np.empty_like(y0)
                st.read(o)
                outs.append(o)
            else:
                o = torch.empty(y0.shape, dtype=torch.float64, device="cuda")
                st.read(o)
                outs.append(o.cpu().numpy())
        info = st.info()
    return y0, outs, info


def run_oracle(w, y0, counts, wd, H, M, checkpoints=False):
    if not checkpoints:
        return [C.advance(w.pde, w.order, y0, counts, wd, H, M)]
    outs, y = [], y0
    for _ in range(M):
        y = C.advance(w.pde, w.order, y, counts, wd, H, 1)
        outs.append(y)
    return outs


# ----------------------------------------------------------------------------- C1 full size
def test_c1_full_every_macro_step(torch_cuda):
    w = get_config("c1")
    counts, wd, H = scheme_for(w)
    y0, g, info = run_gpu(torch_cuda, w, counts, wd, H, w.macro_steps, checkpoints=True)
    o = run_oracle(w, y0, counts, wd, H, w.macro_steps, checkpoints=True)
    for i, (a, b) in enumerate(zip(g, o)):
        assert_parity(a, b, what=f"c1 macro step {i + 1}")
    assert info["substeps_per_macro"] == 24


# ----------------------------------------------------------------------------- reduced, ragged
CASES = [
    # (config, grid (nx, ny, nz), macro steps, weight set)
    ("c1", (200, 1, 1), 20, "square8"),
    ("c1", (77, 1, 1), 10, "square8"),             # odd, single ragged tile
    ("c2", (200, 136, 1), 5, "fallback8"),         # ragged in x (256-wide tiles) and y
    ("c2", (200, 136, 1), 5, "nonzero8"),
    ("c2", (131, 90, 1), 3, "nonzero8"),           # odd nx -> 64-bit path
    ("c3", (264, 200, 1), 3, "nonzero8"),
    ("c3", (520, 72, 1), 2, "fallback8"),
    ("c2", (128, 96, 1), 3, "nonzero8"),           # 2-D TMA kernel (multiple of the 64x16 tile)
    ("c3", (192, 80, 1), 2, "nonzero8"),           # 2-D TMA kernel, FD8
    ("c4", (72, 40, 36), 2, "nonzero8"),           # ragged: 64-wide x tiles, 16-high y tiles
    ("c4", (72, 40, 36), 2, "fallback8"),
    ("c4", (65, 33, 40), 1, "nonzero8"),           # odd nx -> 64-bit path
    ("c5", (70, 34, 48), 1, "nonzero8"),           # {2..16}
    ("c4", (136, 40, 30), 2, "nonzero8"),          # bulk-copy kernel, ragged x tile + wrap split
    ("c5", (128, 48, 36), 1, "nonzero8"),          # TMA kernel (multiple of the 64x16 tile)
    ("c4", (64, 32, 20), 2, "fallback8"),          # TMA kernel, wrap on every halo box
]


@pytest.mark.parametrize("n", [(128, 64, 64), (64, 16, 9), (192, 48, 40), (136, 40, 30)])
def test_bulk_kernel_bitwise_equals_ldg_kernel(torch_cuda, n):
    """The TMA-pipelined kernel (grids that are multiples of its 64x16 tile) and the
    register-prefetch kernel do the same arithmetic in the same order: results must
    agree bit for bit."""
    w = reduced("c4", n, macro_steps=2, weights="nonzero8")
    counts, wd, H = scheme_for(w, "nonzero8")
    _, a, _ = run_gpu(torch_cuda, w, counts, wd, H, 2, opts={"bulk": 1, "fea": 0})   # fea: rounding-level
    _, b, _ = run_gpu(torch_cuda, w, counts, wd, H, 2, opts={"bulk": 0})
    assert np.array_equal(a[0], b[0])


@pytest.mark.parametrize("cfg,n", [("c2", (128, 64, 1)), ("c3", (64, 48, 1)), ("c3", (192, 80, 1)),
                                   ("c2", (64, 16, 1))])
def test_2d_bulk_kernel_bitwise_equals_register_kernel(torch_cuda, cfg, n):
    """2-D acoustics: the TMA-pipelined kernel and the register y-march kernel do the
    same arithmetic in the same order: bit-identical results."""
    w = reduced(cfg, n, macro_steps=2, weights="nonzero8")
    counts, wd, H = scheme_for(w, "nonzero8")
    _, a, _ = run_gpu(torch_cuda, w, counts, wd, H, 2, opts={"bulk": 1})
    _, b, _ = run_gpu(torch_cuda, w, counts, wd, H, 2, opts={"bulk": 0})
    assert np.array_equal(a[0], b[0])


@pytest.mark.parametrize("cfg,n,opts", [("c3", (128, 64, 1), {}), ("c2", (128, 96, 1), {}),
                                        ("c3", (64, 48, 1), {}), ("c3", (192, 96, 1), {"loopback": 2}),
                                        ("c3", (128, 192, 1), {"loopback": 2}),
                                        ("c2", (128, 96, 1), {"loopback": 3, "overlap": 0}),
                                        ("c3", (64, 32, 1), {"graph": 0})])
def test_2d_two_substep_kernels_bitwise_equal_single_steps(torch_cuda, cfg, n, opts):
    """2-D acoustics, two leap-frog substeps per pass (the chain-U and chain-P kernels,
    gbs_acoustic2d_pair.cuh): bit-identical to single-step launches, and the oracle's result."""
    w = reduced(cfg, n, macro_steps=2, weights="nonzero8")
    counts, wd, H = scheme_for(w, "nonzero8")
    y0, a, ia = run_gpu(torch_cuda, w, counts, wd, H, 2, opts=dict(opts, fuse2d=1))
    _, b, ib = run_gpu(torch_cuda, w, counts, wd, H, 2, opts=dict(opts, fuse2d=0))
    assert np.array_equal(a[0], b[0])
    # FE + LF1 + FIN single and (n-2)/2 pairs of two chain kernels: as many stencil launches
    # as substeps, plus (single-slab grids) one ghost-row fill per pair; slabs whose rows are
    # not a multiple of the 32-row band run single substeps
    slab_rows = n[1] // opts.get("loopback", 1)
    if slab_rows % 32 == 0 and opts.get("loopback", 1) == 1:
        assert ia["kernel_launches"] > ib["kernel_launches"]
    else:
        assert ia["kernel_launches"] >= ib["kernel_launches"]
    o = run_oracle(w, y0, counts, wd, H, 2)
    assert_parity(a[0], o[0], what=f"2-D pairs {cfg} {n} {opts}")


@pytest.mark.parametrize("cfg,n", [("c4", (128, 32, 24)), ("c4", (64, 16, 17)), ("c5", (64, 48, 40))])
def test_two_substep_kernel_bitwise_equals_single_steps(torch_cuda, cfg, n):
    """The temporally blocked kernel (two substeps per HBM pass) recomputes the
    intermediate level with the same operations in the same order: bit-identical."""
    w = reduced(cfg, n, macro_steps=2, weights="nonzero8")
    counts, wd, H = scheme_for(w, "nonzero8")
    _, a, ia = run_gpu(torch_cuda, w, counts, wd, H, 2, opts={"fuse": 1, "fea": 0})
    _, b, ib = run_gpu(torch_cuda, w, counts, wd, H, 2, opts={"fuse": 0})
    assert np.array_equal(a[0], b[0])
    S = sum(k + 1 for k in counts)
    assert ib["kernel_launches"] == 2 * S
    # FE + n/2 two-substep passes per sequence; each LF pair as two half launches (option half)
    assert ia["kernel_launches"] == 2 * sum(k for k in counts)


@pytest.mark.parametrize("cfg,n,opts", [
    ("c5", (128, 64, 40), {"half_rpt": 2}),                       # 64 x 32 tiles, 16 warps
    ("c5", (128, 64, 40), {"half_fe": 1}),                        # 64 x 32 tiles, 8 warps, FE too
    ("c4", (64, 48, 30), {}),                                     # ny % 32 != 0: 64 x 16 tiles
    ("c4", (128, 32, 24), {"half_tall": 0}),
    ("c5", (64, 64, 48), {"loopback": 3}),                        # slabs, overlapped exchange
    ("c5", (64, 32, 40), {"loopback": 2, "overlap": 0, "graph": 0}),
    ("c4", (64, 32, 24), {"half_fe": 1, "half_rpt": 2}),          # FE through the half kernel
    ("c5", (64, 32, 40), {"l2hint_half": 0, "zchunk_pair": 7}),   # no cache hints, ragged z chunks
    ("c4", (64, 16, 9), {}),                                      # nz = 2r + 1
])
def test_half_kernels_bitwise_equal_coupled_pair(torch_cuda, cfg, n, opts):
    """Leap-frog pairs as two single-stencil-field launches (gbs_wave3d_half.cuh, option "half"),
    the FE through the same kernel: the same operations in the same order as the coupled pair
    kernel and the FE step kernel -> bit-identical results, and the oracle's within 1e-12."""
    w = reduced(cfg, n, macro_steps=2, weights="nonzero8")
    counts, wd, H = scheme_for(w, "nonzero8")
    y0, a, ia = run_gpu(torch_cuda, w, counts, wd, H, 2, opts=dict(opts, half=1, fea=0))
    _, b, ib = run_gpu(torch_cuda, w, counts, wd, H, 2, opts=dict(opts, half=0, fea=0))
    assert np.array_equal(a[0], b[0])
    slabs = opts.get("loopback", 1)
    pairs = sum(k // 2 - 1 for k in counts)                       # LF pairs per macro step
    # per macro step and slab: one more launch per LF pair (plus, with overlap, its face band)
    per_pair = 1 if (slabs == 1 or not opts.get("overlap", 1)) else 2
    assert ia["kernel_launches"] - ib["kernel_launches"] == 2 * slabs * pairs * per_pair
    o = run_oracle(w, y0, counts, wd, H, 2)
    assert_parity(a[0], o[0], what=f"half kernels {cfg} {n} {opts}")


@pytest.mark.parametrize("cfg,n,opts", [("c5", (128, 64, 40), {}), ("c4", (64, 48, 30), {}),
                                        ("c5", (64, 64, 48), {"loopback": 3}), ("c4", (64, 16, 9), {}),
                                        ("c4", (64, 32, 24), {"loopback": 2, "overlap": 0, "graph": 0})])
def test_fe_fused_with_first_chain_step(torch_cuda, cfg, n, opts):
    _fea_case(torch_cuda, cfg, n, opts)
    # the ring-fed variant of the same pass: the same operations, bit-identical
    w = reduced(cfg, n, macro_steps=2, weights="nonzero8")
    counts, wd, H = scheme_for(w, "nonzero8")
    _, a, _ = run_gpu(torch_cuda, w, counts, wd, H, 2, opts=dict(opts, fea=1, fea_ring=1, fin_ring=1))
    _, b, _ = run_gpu(torch_cuda, w, counts, wd, H, 2, opts=dict(opts, fea=1, fea_ring=0, fin_ring=0))
    assert np.array_equal(a[0], b[0])


def _fea_case(torch_cuda, cfg, n, opts):
    """Option fea: the FE fused with the first step of one leap-frog chain (lap(u_1) by
    linearity, gbs_wave3d_pair.cuh MODE_FEA) -- a rounding-level change, so against the oracle
    and the unfused path within the parity bar, and one launch fewer per sequence with n >= 4."""
    w = reduced(cfg, n, macro_steps=2, weights="nonzero8")
    counts, wd, H = scheme_for(w, "nonzero8")
    y0, a, ia = run_gpu(torch_cuda, w, counts, wd, H, 2, opts=dict(opts, fea=1))
    _, b, ib = run_gpu(torch_cuda, w, counts, wd, H, 2, opts=dict(opts, fea=0))
    o = run_oracle(w, y0, counts, wd, H, 2)
    assert_parity(a[0], o[0], what=f"fea {cfg} {n} {opts}")
    assert_parity(a[0], b[0], what=f"fea vs unfused {cfg} {n} {opts}")
    slabs = opts.get("loopback", 1)
    per = 1 if (slabs == 1 or not opts.get("overlap", 1)) else 2
    assert ib["kernel_launches"] - ia["kernel_launches"] == 2 * slabs * per * sum(1 for k in counts if k >= 4)


@pytest.mark.parametrize("cfg,n,opts", [("c2", (128, 64, 1), {}), ("c3", (192, 96, 1), {}),
                                        ("c2", (64, 48, 1), {"graph": 0}), ("c4", (64, 32, 24), {"fuse": 0})])
def test_two_sequence_streams_bitwise(torch_cuda, cfg, n, opts):
    """Sequences alternating over two CUDA streams (option streams = 2) with the final passes
    kept in ascending n_k order: the same arithmetic and accumulation order -> bit-identical."""
    w = reduced(cfg, n, macro_steps=3, weights="nonzero8")
    counts, wd, H = scheme_for(w, "nonzero8")
    y0, a, _ = run_gpu(torch_cuda, w, counts, wd, H, 3, opts=dict(opts, streams=2))
    _, b, _ = run_gpu(torch_cuda, w, counts, wd, H, 3, opts=dict(opts, streams=1))
    assert np.array_equal(a[0], b[0])
    o = run_oracle(w, y0, counts, wd, H, 3)
    assert_parity(a[0], o[0], what=f"streams=2 {cfg} {n} {opts}")


@pytest.mark.parametrize("opts", [{"band": 1}, {"band": 2}, {"band": 3}, {"l2hint": 0},
                                  {"l2hint": 15, "l2hint_step": 11}])
def test_tile_order_and_cache_policies_do_not_change_results(torch_cuda, opts):
    """The launch order of the 3-D TMA tiles (band; 3 does not divide the 4 x-tiles and falls
    back to whole rows) and the L2 eviction policies move no arithmetic: bit-identical."""
    w = reduced("c5", (256, 32, 20), macro_steps=2, weights="nonzero8")
    counts, wd, H = scheme_for(w, "nonzero8")
    _, a, _ = run_gpu(torch_cuda, w, counts, wd, H, 2, opts=opts)
    _, b, _ = run_gpu(torch_cuda, w, counts, wd, H, 2, opts={})
    assert np.array_equal(a[0], b[0])


@pytest.mark.parametrize("n,steps,wset,M", [((256, 1, 1), (2, 4, 6, 8), "square8", 200),
                                            ((77, 1, 1), (2, 4, 6, 8), "square8", 30),
                                            ((3000, 1, 1), tuple(range(2, 23, 2)), "GBS_8_6", 5)])
def test_cluster_kernel_equals_per_substep_kernels(torch_cuda, n, steps, wset, M):
    """K6: the whole run in one cluster launch (one CTA per sequence, DSMEM combine)
    against the per-substep kernels (bit for bit) and the oracle."""
    w = reduced("c1", n, macro_steps=M).with_(steps=steps, weights=wset)
    counts, ws, _ = W.scheme(wset, steps)
    wd = W.to_double(ws)
    H = S.macro_step_H(w.pde, w.order, w.n, counts, wd)
    y0, a, ia = run_gpu(torch_cuda, w, counts, wd, H, M, opts={"persistent": 1})
    _, b, ib = run_gpu(torch_cuda, w, counts, wd, H, M, opts={"persistent": 0})
    assert ia["kernel_launches"] == 1 and ib["kernel_launches"] == M * sum(k + 1 for k in counts)
    assert np.array_equal(a[0], b[0])
    o = run_oracle(w, y0, counts, wd, H, M)
    assert_parity(a[0], o[0], what="cluster kernel")


@pytest.mark.parametrize("cfg,n,M,wset", CASES)
def test_reduced_every_macro_step(torch_cuda, cfg, n, M, wset):
    w = reduced(cfg, n, macro_steps=M, weights=wset)
    counts, wd, H = scheme_for(w, wset)
    y0, g, _ = run_gpu(torch_cuda, w, counts, wd, H, M, checkpoints=True)
    o = run_oracle(w, y0, counts, wd, H, M, checkpoints=True)
    for i, (a, b) in enumerate(zip(g, o)):
        assert_parity(a, b, what=f"{cfg} {n} {wset} macro step {i + 1}")


# ----------------------------------------------------------------------------- edge cases
@pytest.mark.parametrize("cfg,n,order", [("c4", (9, 9, 9), 8), ("c2", (5, 5, 1), 4),
                                         ("c3", (9, 9, 1), 8), ("c1", (5, 1, 1), 4),
                                         ("c4", (64, 16, 9), 8),     # two-substep TMA path, nz = 2r+1
                                         ("c4", (64, 16, 5), 4),     # FD4 two-substep path, nz = 2r+1
                                         ("c3", (64, 16, 1), 8),     # 2-D TMA path, one 16-row band
                                         ("c2", (64, 16, 1), 4)])
def test_minimum_grid(torch_cuda, cfg, n, order):
    w = reduced(cfg, n, macro_steps=2).with_(order=order)
    counts, wd, H = scheme_for(w)
    y0, g, _ = run_gpu(torch_cuda, w, counts, wd, H, 2)
    o = run_oracle(w, y0, counts, wd, H, 2)
    assert_parity(g[0], o[0], what=f"min grid {n}")


@pytest.mark.parametrize("cfg,n,M", [("c4", (64, 32, 24), 3), ("c5", (64, 48, 40), 2),
                                     ("c3", (192, 80, 1), 3), ("c2", (200, 136, 1), 4)])
def test_optimised_weights_at_their_larger_step(torch_cuda, cfg, n, M):
    """The Appendix-B optimised weights on the config's step counts ("opt8"), run at the H
    their own ISB allows (2.1x / 3.1x the fallback's), through the default kernels
    (two-substep 3-D, TMA 2-D, register 2-D for a ragged grid)."""
    w = reduced(cfg, n, macro_steps=M, weights="opt8")
    counts, wd, H = scheme_for(w)
    c0, w0, H0 = scheme_for(reduced(cfg, n, macro_steps=M))
    assert H > 2.0 * H0
    y0, g, _ = run_gpu(torch_cuda, w, counts, wd, H, M)
    o = run_oracle(w, y0, counts, wd, H, M)
    assert_parity(g[0], o[0], what=f"{cfg} opt8")


@pytest.mark.parametrize("wset,N", [("GBS_8_6", 64), ("GBS_12_8", 64), ("GBS_8_6", 256),
                                    ("GBS_12_8", 128), ("square8", 50), ("GBS_8_8", 32)])
def test_spectral_section41(torch_cuda, wset, N):
    """The paper's own experiment (§4.1): spectral derivative (order 0, circulant
    pairing form in the cluster kernel), IC (1 - cos 2 pi x)/2, lambda = 0.99/pi ISB, one
    period.  Against the oracle (DFT derivative) and the exact solution."""
    import math
    w = get_config("s41").with_(n=(N, 1, 1))
    counts, ws, _ = W.scheme(wset)
    wd = W.to_double(ws)
    M = math.ceil(1.0 / S.macro_step_H("adv1d", 0, w.n, counts, wd, w.h_factor))
    w = w.with_(steps=tuple(counts), weights=wset, macro_steps=M)
    y0, g, info = run_gpu(torch_cuda, w, counts, wd, 1.0 / M, M)
    o = run_oracle(w, y0, counts, wd, 1.0 / M, M)
    assert info["kernel_launches"] == 1
    assert_parity(g[0], o[0], what=f"s41 {wset} N={N}")
    err_gpu = np.max(np.abs(g[0] - y0))
    err_or = np.max(np.abs(o[0] - y0))
    assert err_gpu <= 1.01 * err_or + 1e-13


@pytest.mark.parametrize("wset,N,opts", [("GBS_8_6", 64, {"persistent": 0}), ("GBS_12_8", 256, {"persistent": 0}),
                                          ("square8", 8192, {}), ("square8", 6402, {"graph": 0})])
def test_spectral_fft_path(torch_cuda, wset, N, opts):
    """The spectral derivative beyond the cluster kernel (N > 6400, or option persistent=0):
    cuFFT D2Z, multiplication by i 2 pi k (Nyquist dropped), Z2D, then the pointwise substep
    update -- against the oracle's DFT derivative, the section 4.1 IC and H rule."""
    import math
    w = get_config("s41").with_(n=(N, 1, 1))
    counts, ws, _ = W.scheme(wset)
    wd = W.to_double(ws)
    H = 1.0 / math.ceil(1.0 / S.macro_step_H("adv1d", 0, w.n, counts, wd, w.h_factor))
    M = 3
    w = w.with_(steps=tuple(counts), weights=wset, macro_steps=M)
    y0, g, info = run_gpu(torch_cuda, w, counts, wd, H, M, opts=opts)
    o = run_oracle(w, y0, counts, wd, H, M)
    assert info["kernel_launches"] == 2 * M * sum(k + 1 for k in counts)   # per substep: ik scale + update
    assert_parity(g[0], o[0], what=f"spectral fft {wset} N={N}")


def test_spectral_fft_large_grid_against_exact_solution(torch_cuda):
    """N = 2^20 (far beyond the cluster kernel): the section 4.1 IC (1 - cos 2 pi x)/2 is one
    Fourier mode, which the spectral derivative resolves exactly, so after M macro steps the
    result is (1 - Re(R(H lambda)^M e^{2 pi i x}))/2 with lambda = -2 pi i -- the closed form
    of the scheme's stability polynomial (oracle/stability.py), no O(N^2) oracle run."""
    import math
    N = 1 << 20
    w = get_config("s41").with_(n=(N, 1, 1))
    counts, ws, _ = W.scheme("GBS_8_6")
    wd = W.to_double(ws)
    H = 1.0 / math.ceil(1.0 / S.macro_step_H("adv1d", 0, w.n, counts, wd, w.h_factor))
    M = 3
    w = w.with_(steps=tuple(counts), weights="GBS_8_6", macro_steps=M)
    y0, g, _ = run_gpu(torch_cuda, w, counts, wd, H, M)
    amp = complex(S.R_eval(counts, wd, np.array([complex(0.0, -2.0 * math.pi * H)]))[0]) ** M
    x = np.arange(N) / N
    exact = 0.5 * (1.0 - (amp * np.exp(2j * math.pi * x)).real)
    assert_parity(g[0], exact[None, :], what="spectral fft N=2^20 vs closed form")


def test_single_sequence_and_fd4_wave(torch_cuda):
    w = reduced("c4", (24, 20, 18), macro_steps=3).with_(order=4, steps=(2,))
    y0 = make_ic(w)
    H = 1e-3
    _, g, _ = run_gpu(torch_cuda, w, [2], [1.0], H, 3)
    o = run_oracle(w, y0, [2], [1.0], H, 3)
    assert_parity(g[0], o[0], what="m=1")


def test_paper_scheme_gbs86(torch_cuda):
    """GBS_8,6, 11 sequences, on a 3-D wave grid."""
    w = reduced("c4", (34, 30, 28), macro_steps=2).with_(steps=tuple(range(2, 23, 2)),
                                                          weights="GBS_8_6")
    counts, ws, _ = W.scheme("GBS_8_6")
    wd = W.to_double(ws)
    H = S.macro_step_H(w.pde, w.order, w.n, counts, wd)
    y0, g, info = run_gpu(torch_cuda, w, counts, wd, H, 2)
    o = run_oracle(w, y0, counts, wd, H, 2)
    assert_parity(g[0], o[0], what="GBS_8_6")
    assert info["substeps_per_macro"] == sum(n + 1 for n in counts)


@pytest.mark.parametrize("wset", ["GBS_8_6", "GBS_8_8", "GBS_12_8", "FD12"])
def test_paper_schemes_on_the_two_substep_path(torch_cuda, wset):
    """The paper's printed schemes (§3.3, §3.8: 6-15 sequences, n_k up to 30, order
    8 and 12) through the default 3-D path (TMA grid: FE + two-substep launches), against the
    oracle, at each scheme's own H = 0.5 ISB / rho."""
    counts, ws, _ = W.scheme(wset)
    wd = W.to_double(ws)
    w = reduced("c4", (64, 32, 24), macro_steps=2).with_(steps=tuple(counts), weights=wset)
    H = S.macro_step_H(w.pde, w.order, w.n, counts, wd)
    y0, g, info = run_gpu(torch_cuda, w, counts, wd, H, 2)
    o = run_oracle(w, y0, counts, wd, H, 2)
    assert_parity(g[0], o[0], what=wset)
    # FE fused with chain A's first step (n >= 4), the other half launches, LF+FIN
    assert info["kernel_launches"] == 2 * sum(n - (1 if n >= 4 else 0) for n in counts)


def test_host_buffers_match_device_buffers(torch_cuda):
    w = reduced("c2", (96, 64, 1), macro_steps=2, weights="nonzero8")
    counts, wd, H = scheme_for(w, "nonzero8")
    _, gd, _ = run_gpu(torch_cuda, w, counts, wd, H, 2)
    _, gh, _ = run_gpu(torch_cuda, w, counts, wd, H, 2, host=True)
    assert np.array_equal(gd[0], gh[0])


def test_slab_io_round_trip(torch_cuda):
    """gbs_write_slab / gbs_read_slab (one GPU: the slab is the whole grid, also with
    loopback slabs) move the same bytes as the full-grid calls."""
    gbs = gbs_mod()
    torch = torch_cuda
    w = reduced("c4", (64, 32, 24), macro_steps=1, weights="nonzero8")
    counts, wd, H = scheme_for(w, "nonzero8")
    y0 = make_ic(w)
    outs = []
    for lb in (1, 3):
        with gbs.Stepper(w.pde, w.n, w.order, counts, wd, loopback=lb) as st:
            st.write_slab(torch.from_numpy(y0).cuda())
            st.advance(1, H)
            a = torch.empty(y0.shape, dtype=torch.float64, device="cuda")
            b = np.empty_like(y0)
            st.read_slab(a)
            st.read(b)
            assert np.array_equal(a.cpu().numpy(), b)
            outs.append(b)
    assert np.array_equal(outs[0], outs[1])


@pytest.mark.parametrize("cfg,n,lb", [("c4", (64, 32, 24), 1), ("c4", (64, 32, 24), 3),
                                      ("c3", (128, 64, 1), 2), ("c1", (256, 1, 1), 1)])
def test_async_io_pipeline(torch_cuda, cfg, n, lb):
    """gbs_write_slab_async / gbs_read_slab_async: a write-advance-read loop of several steps
    with distinct inputs (host and device buffers) returns, bit for bit, what the synchronous
    calls return step by step."""
    gbs = gbs_mod()
    torch = torch_cuda
    w = reduced(cfg, n, macro_steps=1, weights="nonzero8" if cfg != "c1" else None)
    counts, wd, H = scheme_for(w, "nonzero8" if cfg != "c1" else None)
    y0 = make_ic(w)
    ins = [y0 * (1.0 + 0.25 * k) for k in range(4)]
    ref = []
    with gbs.Stepper(w.pde, w.n, w.order, counts, wd, loopback=lb) as st:
        for x in ins:
            st.write_slab(x)
            st.advance(2, H)
            o = np.empty_like(x)
            st.read_slab(o)
            ref.append(o)
    for on_dev in (False, True):
        with gbs.Stepper(w.pde, w.n, w.order, counts, wd, loopback=lb) as st:
            if on_dev:
                src = [torch.from_numpy(x).cuda() for x in ins]
                outs = [torch.empty(x.shape, dtype=torch.float64, device="cuda") for x in ins]
            else:
                src = [torch.from_numpy(x).pin_memory() for x in ins]
                outs = [torch.empty(x.shape, dtype=torch.float64).pin_memory() for x in ins]
            for x, o in zip(src, outs):
                st.write_async(x)
                st.advance(2, H)
                st.read_async(o)
            st.sync()
            for o, r in zip(outs, ref):
                assert np.array_equal(o.cpu().numpy(), r)


@pytest.mark.parametrize("cfg,n,lb", [("c4", (64, 32, 24), 1), ("c5", (64, 48, 40), 2), ("c3", (128, 64, 1), 1),
                                      ("c2", (200, 136, 1), 2)])
def test_torch_owned_workspace(torch_cuda, cfg, n, lb):
    """State buffers carved from a torch tensor (gbs_bind_workspace): same bytes as the
    context's own allocation; the tensor really is the state memory (the bytes grow by
    exactly gbs_workspace_bytes), and rebinding discards the state."""
    gbs = gbs_mod()
    torch = torch_cuda
    w = reduced(cfg, n, macro_steps=2, weights="nonzero8")
    counts, wd, H = scheme_for(w, "nonzero8")
    _, a, _ = run_gpu(torch, w, counts, wd, H, 2, opts={"loopback": lb})
    y0 = make_ic(w)
    before = torch.cuda.memory_allocated()
    with gbs.Stepper(w.pde, w.n, w.order, counts, wd, torch_memory=True, loopback=lb) as st:
        nbytes = gbs.gbs_workspace_bytes(st.ctx)
        assert torch.cuda.memory_allocated() - before >= nbytes > 0
        st.write(y0)
        st.advance(2, H)
        out = np.empty_like(y0)
        st.read(out)
        assert np.array_equal(out, a[0])
        gbs.gbs_bind_workspace(st.ctx, None)           # back to own buffers: state discarded
        with pytest.raises(gbs.GbsError) as e:
            st.advance(1, H)
        assert e.value.code == gbs.GBS_E_STATE
        small = torch.empty(16, dtype=torch.uint8, device="cuda")
        with pytest.raises(gbs.GbsError) as e:
            gbs.gbs_bind_workspace(st.ctx, small)
        assert e.value.code == gbs.GBS_E_INVAL


def test_graph_replay_is_bitwise_identical(torch_cuda):
    w = reduced("c4", (40, 36, 34), macro_steps=3, weights="nonzero8")
    counts, wd, H = scheme_for(w, "nonzero8")
    _, a, ia = run_gpu(torch_cuda, w, counts, wd, H, 3, opts={"graph": 1})
    _, b, ib = run_gpu(torch_cuda, w, counts, wd, H, 3, opts={"graph": 0})
    assert ia["uses_graph"] == 1 and ib["uses_graph"] == 0
    assert np.array_equal(a[0], b[0])
    assert ia["kernel_launches"] == ib["kernel_launches"] == 3 * 48


@pytest.mark.parametrize("cfg,n,slabs", [("c4", (64, 16, 16), 4),      # slabs exactly r planes thick
                                         ("c4", (40, 36, 32), 2), ("c4", (40, 36, 32), 4),
                                         ("c4", (128, 32, 36), 3), ("c5", (64, 32, 32), 4),
                                         ("c5", (36, 20, 24), 3), ("c2", (96, 64, 1), 4),
                                         ("c3", (80, 48, 1), 3), ("c2", (128, 64, 1), 4),
                                         ("c3", (64, 96, 1), 3)])
def test_loopback_slabs(torch_cuda, cfg, n, slabs):
    """z-slabs (y in 2-D) with ghost planes and halo copies, emulated on one GPU."""
    w = reduced(cfg, n, macro_steps=2, weights="nonzero8")
    counts, wd, H = scheme_for(w, "nonzero8")
    y0, g, info = run_gpu(torch_cuda, w, counts, wd, H, 2, opts={"loopback": slabs})
    o = run_oracle(w, y0, counts, wd, H, 2)
    assert info["slabs"] == slabs
    assert_parity(g[0], o[0], what=f"loopback {slabs}")


@pytest.mark.parametrize("cfg,n,slabs", [("c4", (64, 32, 48), 2), ("c5", (64, 48, 60), 3),
                                         ("c4", (40, 36, 36), 3), ("c2", (128, 96, 1), 2),
                                         ("c3", (200, 72, 1), 3)])
def test_halo_overlap_is_bitwise_identical(torch_cuda, cfg, n, slabs):
    """Slabbed layouts exchange the halo on a comm stream while the interior planes are
    computed, then compute the face bands (option overlap, default on): the same bytes as
    exchanging first, with and without graph capture, and the oracle's result."""
    w = reduced(cfg, n, macro_steps=2, weights="nonzero8")
    counts, wd, H = scheme_for(w, "nonzero8")
    y0, a, _ = run_gpu(torch_cuda, w, counts, wd, H, 2, opts={"loopback": slabs, "overlap": 1})
    _, b, _ = run_gpu(torch_cuda, w, counts, wd, H, 2, opts={"loopback": slabs, "overlap": 0})
    _, c, _ = run_gpu(torch_cuda, w, counts, wd, H, 2, opts={"loopback": slabs, "overlap": 1, "graph": 0})
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[0], c[0])
    o = run_oracle(w, y0, counts, wd, H, 2)
    assert_parity(a[0], o[0], what=f"overlap {cfg} {slabs} slabs")


@pytest.mark.parametrize("cfg,n,slabs,overlap", [("c4", (64, 32, 48), 2, 1), ("c5", (64, 48, 60), 3, 1),
                                                 ("c4", (40, 36, 36), 3, 0), ("c5", (64, 16, 24), 2, 0),
                                                 ("c3", (200, 72, 1), 3, 1), ("c2", (128, 96, 1), 2, 0)])
def test_loopback_halos_through_nccl(torch_cuda, cfg, n, slabs, overlap):
    """The multi-GPU transfer path on one GPU: the loopback slabs' ghost planes move by grouped
    ncclSend / ncclRecv on a one-rank communicator (option loopback_nccl; eager launches, halo
    on the comm stream under overlap) -- the same bytes as the device-copy loopback."""
    w = reduced(cfg, n, macro_steps=2, weights="nonzero8")
    counts, wd, H = scheme_for(w, "nonzero8")
    y0, a, _ = run_gpu(torch_cuda, w, counts, wd, H, 2,
                       opts={"loopback": slabs, "overlap": overlap, "loopback_nccl": 1})
    _, b, _ = run_gpu(torch_cuda, w, counts, wd, H, 2, opts={"loopback": slabs, "overlap": overlap})
    assert np.array_equal(a[0], b[0])
    o = run_oracle(w, y0, counts, wd, H, 2)
    assert_parity(a[0], o[0], what=f"nccl loopback {cfg} {slabs} slabs")


@pytest.mark.parametrize("cfg,n,slabs", [("c5", (64, 32, 48), 2), ("c4", (64, 16, 36), 3), ("c5", (128, 32, 64), 4),
                                         ("c4", (64, 16, 16), 4), ("c5", (64, 48, 60), 3)])
def test_peer_halo_pushes_match_exchange(torch_cuda, cfg, n, slabs):
    """Peer pushes (option peer, loopback slabs): the FE and two-substep kernels store their
    face planes into the neighbouring slabs' ghost planes and order themselves by epoch flags
    -- no halo exchange.  Bit-identical to the exchanged loopback and to the single slab, and
    the oracle's result; a second advance continues from the pushed ghosts."""
    w = reduced(cfg, n, macro_steps=2, weights="nonzero8")
    counts, wd, H = scheme_for(w, "nonzero8")
    y0, a, ia = run_gpu(torch_cuda, w, counts, wd, H, 2, opts={"loopback": slabs, "peer": 1})
    # (peer pushes run the coupled pair kernel: compare launch counts with half = 0)
    _, b, ib = run_gpu(torch_cuda, w, counts, wd, H, 2, opts={"loopback": slabs, "overlap": 0, "half": 0})
    _, c1, _ = run_gpu(torch_cuda, w, counts, wd, H, 2, opts={"fea": 0})
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[0], c1[0])
    # one stencil launch + one epoch signal per slab per substep launch, no exchange
    assert ia["kernel_launches"] == 2 * ib["kernel_launches"]
    _, d, _ = run_gpu(torch_cuda, w, counts, wd, H, 2, checkpoints=True, opts={"loopback": slabs, "peer": 1})
    assert np.array_equal(d[-1], a[0])
    o = run_oracle(w, y0, counts, wd, H, 2)
    assert_parity(a[0], o[0], what=f"peer {cfg} {n} {slabs}")


def test_peer_option_rejected_where_it_does_not_apply(torch_cuda):
    gbs = gbs_mod()
    w = reduced("c4", (40, 36, 32), macro_steps=1, weights="nonzero8")   # not whole 64x16 tiles
    counts, wd, _ = scheme_for(w, "nonzero8")
    with gbs.Stepper(w.pde, w.n, w.order, counts, wd, loopback=2) as st:
        with pytest.raises(gbs.GbsError) as e:
            gbs.gbs_set_option(st.ctx, "peer", 1)
        assert e.value.code == gbs.GBS_E_UNSUPPORTED
        with pytest.raises(gbs.GbsError) as e:
            gbs.gbs_bind_peers(st.ctx, 1 << 40, 1 << 40)      # one GPU: not a multi-GPU slab layout
        assert e.value.code in (gbs.GBS_E_STATE, gbs.GBS_E_UNSUPPORTED)


# ----------------------------------------------------------------------------- errors
def test_error_paths(torch_cuda):
    gbs = gbs_mod()
    ctx = gbs.gbs_create("wave3d", (16, 16, 16), 8, [2, 4], [-1 / 3, 4 / 3])
    try:
        with pytest.raises(gbs.GbsError) as e:
            gbs.gbs_advance(ctx, 1, 1e-3)
        assert e.value.code == gbs.GBS_E_STATE
        y = torch_cuda.zeros((2, 16, 16, 16), dtype=torch_cuda.float64, device="cuda")
        gbs.gbs_write_state(ctx, y)
        for H in (0.0, -1.0, float("inf"), float("nan")):
            with pytest.raises(gbs.GbsError) as e:
                gbs.gbs_advance(ctx, 1, H)
            assert e.value.code == gbs.GBS_E_INVAL
        with pytest.raises(gbs.GbsError) as e:
            gbs.gbs_read_state(ctx, torch_cuda.zeros(10, dtype=torch_cuda.float64, device="cuda"))
        assert e.value.code == gbs.GBS_E_INVAL
        with pytest.raises(gbs.GbsError):
            gbs.gbs_set_option(ctx, "no_such_option", 1)
    finally:
        gbs.gbs_destroy(ctx)


def test_instability_is_reported(torch_cuda):
    """H far beyond the ISB: the extreme mode overflows and GBS_E_NONFINITE surfaces."""
    gbs = gbs_mod()
    n = 16
    x = np.arange(n) / n
    z, yy, xx = np.meshgrid(x, x, x, indexing="ij")
    u = np.cos(np.pi * n * xx) * np.cos(np.pi * n * yy) * np.cos(np.pi * n * z)
    y0 = np.stack([u, np.zeros_like(u)])
    counts, ws, _ = W.scheme("square8")
    wd = W.to_double(ws)
    H = 3.0 * S.isb(counts, wd) / S.rho("wave3d", 8, (n, n, n))
    with gbs.Stepper("wave3d", (n, n, n), 8, counts, wd) as st:
        st.write(torch_cuda.from_numpy(y0).cuda())
        st.advance(400, H)
        with pytest.raises(gbs.GbsError) as e:
            st.read(torch_cuda.empty((2, n, n, n), dtype=torch_cuda.float64, device="cuda"))
        assert e.value.code == gbs.GBS_E_NONFINITE


# ----------------------------------------------------------------------------- full sizes
def _sample_boxes(w, y0, counts, wd, H, centres):
    """Oracle values at sampled points after ONE macro step, each from a periodically
    extracted box of half-width r*(max n_k + 1) (bitwise equal to the full-grid oracle,
    tests/test_oracle_stepping.py::test_box_sample_reproduces_full_grid_value_bitwise)."""
    R = (w.order // 2) * (max(counts) + 1)
    nx, ny, nz = w.n
    vals = []
    for c in centres:
        if w.ndim == 3:
            cz, cy, cx = c
            iz = np.arange(cz - R, cz + R + 1) % nz
            iy = np.arange(cy - R, cy + R + 1) % ny
            ix = np.arange(cx - R, cx + R + 1) % nx
            box = np.ascontiguousarray(y0[:, iz][:, :, iy][:, :, :, ix])
            out = C.advance(w.pde, w.order, box, counts, wd, H, 1, scale=w.n)
            vals.append(out[:, R, R, R])
        else:
            cy, cx = c
            iy = np.arange(cy - R, cy + R + 1) % ny
            ix = np.arange(cx - R, cx + R + 1) % nx
            box = np.ascontiguousarray(y0[:, iy][:, :, ix])
            out = C.advance(w.pde, w.order, box, counts, wd, H, 1, scale=w.n)
            vals.append(out[:, R, R])
    return np.array(vals)


@pytest.mark.slow
@pytest.mark.parametrize("cfg", ["c2", "c3"])
def test_2d_full_size_whole_run(torch_cuda, cfg):
    """The whole BASELINE.json run (C2: 1024^2, 50 macro steps; C3: 4096^2, 20) against the
    oracle, checked every 10 macro steps over the full state."""
    w = get_config(cfg)
    counts, wd, H = scheme_for(w)
    gbs = gbs_mod()
    torch = torch_cuda
    y0 = make_ic(w)
    ref = y0
    with gbs.Stepper(w.pde, w.n, w.order, counts, wd) as st:
        st.write(torch.from_numpy(y0).cuda())
        done = 0
        while done < w.macro_steps:
            k = min(10, w.macro_steps - done)
            st.advance(k, H)
            out = torch.empty(y0.shape, dtype=torch.float64, device="cuda")
            st.read(out)
            ref = C.advance(w.pde, w.order, ref, counts, wd, H, k)
            done += k
            assert_parity(out.cpu().numpy(), ref, what=f"{cfg} full, macro step {done}")


@pytest.mark.slow
@pytest.mark.parametrize("cfg,M", [("c2", 10), ("c3", 4)])
def test_2d_full_size_nonzero_weights(torch_cuda, cfg, M):
    """C2 / C3 at full size with the all-nonzero parity weights (fallback8 gives the
    sequences 10 and 12 weight 0, so only a nonzero set shows a bug in them), full state."""
    w = get_config(cfg).with_(weights="nonzero8")
    counts, wd, H = scheme_for(get_config(cfg), "nonzero8")
    gbs = gbs_mod()
    y0 = make_ic(w)
    with gbs.Stepper(w.pde, w.n, w.order, counts, wd) as st:
        st.write(torch_cuda.from_numpy(y0).cuda())
        st.advance(M, H)
        out = np.empty_like(y0)
        st.read(out)
    ref = C.advance(w.pde, w.order, y0, counts, wd, H, M)
    assert_parity(out, ref, what=f"{cfg} full nonzero8, {M} macro steps")


@pytest.mark.slow
def test_c4_full_size_whole_run(torch_cuda):
    """The whole BASELINE.json C4 run (512^3, FD8, {2..12}, 10 macro steps; the two-substep
    TMA path) against the oracle over the full state after 5 and 10 macro steps (the oracle
    takes about two minutes on the GPU box's host cores)."""
    w = get_config("c4")
    counts, wd, H = scheme_for(w)
    gbs = gbs_mod()
    torch = torch_cuda
    y0 = make_ic(w)
    ref = y0
    with gbs.Stepper(w.pde, w.n, w.order, counts, wd) as st:
        st.write(torch.from_numpy(y0).cuda())
        for done in (5, 10):
            st.advance(5, H)
            out = np.empty_like(y0)
            st.read(out)
            ref = C.advance(w.pde, w.order, ref, counts, wd, H, 5)
            assert_parity(out, ref, what=f"c4 full, macro step {done}")


@pytest.mark.slow
def test_c4_full_size_whole_run_nonzero_weights(torch_cuda):
    """The whole C4 run (512^3, 10 macro steps) with the all-nonzero parity weights (SURVEY S3:
    with fallback8 the sequences 10 and 12 carry w = 0, so a bug in them would be invisible)."""
    w = get_config("c4").with_(weights="nonzero8")
    counts, wd, H = scheme_for(get_config("c4"), "nonzero8")
    gbs = gbs_mod()
    y0 = make_ic(w)
    with gbs.Stepper(w.pde, w.n, w.order, counts, wd) as st:
        st.write(torch_cuda.from_numpy(y0).cuda())
        st.advance(w.macro_steps, H)
        out = np.empty_like(y0)
        st.read(out)
    ref = C.advance(w.pde, w.order, y0, counts, wd, H, w.macro_steps)
    assert_parity(out, ref, what="c4 full nonzero8, 10 macro steps")


def _host_ram_gib():
    try:
        import psutil
        return psutil.virtual_memory().total / 2**30
    except Exception:
        return 0.0


@pytest.mark.slow
@pytest.mark.parametrize("wset", ["nonzero8", "fallback8"])
def test_c5_scheme_full_state_at_bench_geometry(torch_cuda, wset):
    """C5's scheme ({2..16}, FD8) over the WHOLE state of a 1024 x 1024 x nz grid in the bench's
    launch geometry: the two-substep TMA kernel with 256-plane z-chunks (the automatic choice at
    C5; forced here), 1024 x-y tiles per chunk.  nz = 512 (two chunks per column, 13.8 waves of
    CTAs on 148 SMs) when the host has the RAM for the oracle, else 256.  One macro step = 80
    substeps, 8 sequences, the C5 FE / LF-pair / LF+FIN0 / LF+FINACC launches."""
    nz = 512 if _host_ram_gib() >= 160 else 256
    w = get_config("c5").with_(n=(1024, 1024, nz), weights=wset)
    counts, wd, H = scheme_for(get_config("c5"), wset)
    gbs = gbs_mod()
    y0 = make_ic(w)
    with gbs.Stepper(w.pde, w.n, w.order, counts, wd, zchunk_pair=256) as st:
        st.write(torch_cuda.from_numpy(y0).cuda())
        st.advance(1, H)
        out = np.empty_like(y0)
        st.read(out)
        launches = st.info()["kernel_launches"]
    # FE fused with chain A's first step (n >= 4), the other halves, LF+FIN
    assert launches == sum(k - (1 if k >= 4 else 0) for k in counts)
    ref = C.advance(w.pde, w.order, y0, counts, wd, H, 1)
    assert_parity(out, ref, what=f"c5 scheme 1024x1024x{nz} {wset}, one macro step, 256-plane chunks")


@pytest.mark.slow
def test_c5_whole_run_conserves_means(torch_cuda):
    """Property at full size: the whole C5 run (1024^3, 4 macro steps). The zero Fourier mode
    of the 3-D wave evolves as u0' = v0, v0' = 0 with R(0)=1, R'(0)=sum w = 1, so the means of
    u and v after M macro steps are mean(u) + M H mean(v) and mean(v) (to rounding)."""
    torch = torch_cuda
    gbs = gbs_mod()
    w = get_config("c5")
    counts, wd, H = scheme_for(w)
    y0 = make_ic(w)
    mu0, mv0 = float(y0[0].mean()), float(y0[1].mean())
    with gbs.Stepper(w.pde, w.n, w.order, counts, wd) as st:
        st.write(torch.from_numpy(y0).cuda())
        st.advance(w.macro_steps, H)
        out = torch.empty(y0.shape, dtype=torch.float64, device="cuda")
        st.read(out)
        mu, mv = float(out[0].mean()), float(out[1].mean())
        rms = float(out[0].pow(2).mean().sqrt())
        assert torch.isfinite(out).all()
    assert abs(mu - (mu0 + w.macro_steps * H * mv0)) < 1e-12 and abs(mv - mv0) < 1e-12
    assert 0.1 < rms < 10.0


@pytest.mark.slow
@pytest.mark.parametrize("cfg,wset", [("c4", None), ("c5", None), ("c5", "nonzero8")])
def test_3d_full_size_sampled(torch_cuda, cfg, wset):
    torch = torch_cuda
    gbs = gbs_mod()
    w = get_config(cfg)
    counts, wd, H = scheme_for(w, wset)
    y0 = make_ic(w)
    nx, ny, nz = w.n
    rng = np.random.default_rng(7)
    centres = [(0, 0, 0), (nz - 1, ny - 1, nx - 1), (nz // 2, 0, nx - 1), (3, ny // 3, 5)]
    centres += [tuple(int(v) for v in rng.integers(0, [nz, ny, nx])) for _ in range(4)]
    with gbs.Stepper(w.pde, w.n, w.order, counts, wd) as st:
        st.write(torch.from_numpy(y0).cuda())
        st.advance(1, H)
        out = torch.empty(y0.shape, dtype=torch.float64, device="cuda")
        st.read(out)
        idx = torch.tensor(centres, device="cuda")
        got = out[:, idx[:, 0], idx[:, 1], idx[:, 2]].T.cpu().numpy()
        del out
    ref = _sample_boxes(w, y0, counts, wd, H, centres)
    scale = np.sqrt(np.mean(y0 * y0))          # RMS of the input (|R| <= 1: norms do not grow)
    err = np.max(np.abs(got - ref)) / scale
    assert err <= TOL, f"{cfg}: max |gpu - oracle| / rms = {err:.3e}"


# ----------------------------------------------------------------------------- randomized
def _random_cases(seed=20261020, count=14, include_1d=False):
    """Seeded random small cases: PDE, grid (TMA-sized or ragged), slab count and options.
    Every case is checked against the oracle, so a bug in any launch variant (register / TMA /
    two-substep kernels, slabs, overlap split, face-band launch, graphs, tile order) shows."""
    rng = np.random.default_rng(seed)
    cases = []
    while len(cases) < count:
        cfg = str(rng.choice(["c1", "c2", "c3", "c4", "c5"] if include_1d else ["c2", "c3", "c4", "c5"]))
        if cfg == "c1":
            cases.append((cfg, (int(rng.integers(9, 700)), 1, 1),
                          {"persistent": int(rng.integers(0, 2)), "graph": int(rng.integers(0, 2))}))
            continue
        if cfg in ("c4", "c5"):
            nx = int(rng.choice([64, 128, 40, 72]))
            ny = int(rng.choice([16, 32, 36]))
            nz = int(rng.choice([16, 24, 30, 48]))
            n = (nx, ny, nz)
            slow = nz
        else:
            nx = int(rng.choice([64, 128, 96, 200]))
            ny = int(rng.choice([32, 48, 64, 96, 72]))
            n = (nx, ny, 1)
            slow = ny
        R = 4 if cfg in ("c3", "c4", "c5") else 2
        lbs = [s for s in (1, 2, 3, 4) if slow % s == 0 and slow // s >= R]
        lb = int(rng.choice(lbs))
        opts = {"loopback": lb, "overlap": int(rng.integers(0, 2)), "graph": int(rng.integers(0, 2)),
                "half": int(rng.integers(0, 2)), "half_rpt": int(rng.choice([2, 4])),
                "fea": int(rng.integers(0, 2)), "streams": int(rng.choice([1, 1, 2])),
                "fuse": int(rng.integers(0, 2)), "band": int(rng.choice([0, 1, 2])),
                "zchunk": int(rng.choice([0, 0, 8, 17])), "zchunk_pair": int(rng.choice([0, 0, 5, 32])),
                "l2hint": int(rng.choice([11, 0, 15]))}
        if cfg in ("c2", "c3"):
            opts["fuse2d"] = int(rng.integers(0, 2))
        if lb > 1 and rng.integers(0, 4) == 0:
            opts["loopback_nccl"] = 1
        if (cfg in ("c4", "c5") and lb > 1 and n[0] % 64 == 0 and n[1] % 16 == 0 and opts["fuse"]
                and rng.integers(0, 2) == 0):
            opts["peer"] = 1
        cases.append((cfg, n, opts))
    return cases


@pytest.mark.parametrize("cfg,n,opts", _random_cases())
def test_randomized_launch_variants_match_oracle(torch_cuda, cfg, n, opts):
    wset = "square8" if cfg == "c1" else "nonzero8"
    w = reduced(cfg, n, macro_steps=2, weights=wset)
    counts, wd, H = scheme_for(w, wset)
    y0, g, _ = run_gpu(torch_cuda, w, counts, wd, H, 2, opts=opts)
    o = run_oracle(w, y0, counts, wd, H, 2)
    assert_parity(g[0], o[0], what=f"{cfg} {n} {opts}")

"""The C-ABI library: it loads, exports every symbol include/gbs.h declares, and
refuses to run without a GPU (no CPU fallback).  No compute calls here."""

import ctypes
import os
import re
import subprocess

import pytest

from conftest import ROOT
from paper_1907_11771_b200 import _build, gbs


def header_symbols():
    src = open(os.path.join(ROOT, "include", "gbs.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gbs_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    _build.build()
    return gbs.load()


def test_header_declares_the_boundary():
    syms = header_symbols()
    for s in ("gbs_create", "gbs_advance", "gbs_read_state", "gbs_write_state", "gbs_destroy"):
        assert s in syms
    assert sorted(gbs.EXPORTS) == syms


def test_library_exports_every_declared_symbol(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", _build.LIB], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (gbs_[a-z0-9_]+)", out))
    missing = [s for s in header_symbols() if s not in exported]
    assert not missing, missing
    for s in header_symbols():
        assert hasattr(lib, s)


def test_only_abi_symbols_are_exported(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", _build.LIB], capture_output=True,
                         text=True, check=True).stdout
    ours = [l.split()[-1] for l in out.splitlines() if " T " in l]
    assert all(s.startswith("gbs_") for s in ours), ours


def test_library_is_sm100a(lib):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _build.LIB],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_strerror(lib):
    assert gbs.gbs_strerror(gbs.GBS_E_WEIGHTS) == "invalid extrapolation weights"
    assert gbs.gbs_strerror(0) == "ok"


def test_create_without_gpu_fails_loudly(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(gbs.GbsError) as e:
        gbs.gbs_create("wave3d", (16, 16, 16), 8, [2, 4], [-1 / 3, 4 / 3], stream=0)
    assert e.value.code == gbs.GBS_E_CUDA


def test_null_context_calls_fail_cleanly(lib):
    """Every entry point taking a context rejects NULL with GBS_E_INVAL (no crash, no GPU)."""
    import ctypes
    L = gbs.load()
    buf = (ctypes.c_double * 4)()
    for fn in ("gbs_write_state", "gbs_read_state", "gbs_write_slab", "gbs_read_slab",
               "gbs_write_slab_async", "gbs_read_slab_async"):
        assert getattr(L, fn)(None, ctypes.cast(buf, ctypes.c_void_p), 4, 0) == gbs.GBS_E_INVAL, fn
    assert L.gbs_advance(None, 1, 1e-3) == gbs.GBS_E_INVAL
    assert L.gbs_sync(None) == gbs.GBS_E_INVAL
    L.gbs_destroy(None)                     # no-op


def test_argument_validation_precedes_device(lib):
    """Invalid arguments are rejected with the documented codes even without a GPU."""
    cases = [
        (("wave3d", (16, 16, 16), 6, [2, 4], [-1 / 3, 4 / 3]), gbs.GBS_E_INVAL),   # order 6
        (("wave3d", (16, 16, 16), 8, [2, 3], [-1 / 3, 4 / 3]), gbs.GBS_E_INVAL),   # odd n_k
        (("wave3d", (16, 16, 16), 8, [4, 4], [-1 / 3, 4 / 3]), gbs.GBS_E_INVAL),   # duplicate
        (("wave3d", (8, 16, 16), 8, [2, 4], [-1 / 3, 4 / 3]), gbs.GBS_E_INVAL),    # n < 2r+1
        (("wave3d", (16, 16, 16), 8, [2, 4], [0.5, 0.6]), gbs.GBS_E_WEIGHTS),      # sum != 1
        (("wave3d", (16, 16, 16), 8, [2, 4], [float("nan"), 1.0]), gbs.GBS_E_WEIGHTS),
        (("acoustic2d", (16, 16, 16), 4, [2, 4], [-1 / 3, 4 / 3]), gbs.GBS_E_INVAL),  # nz != 1
        (("wave3d", (16, 16, 16), 0, [2, 4], [-1 / 3, 4 / 3]), gbs.GBS_E_INVAL),   # spectral: 1-D only
        (("adv1d", (63, 1, 1), 0, [2, 4], [-1 / 3, 4 / 3]), gbs.GBS_E_INVAL),      # spectral: even N
        (("adv1d", (2, 1, 1), 0, [2, 4], [-1 / 3, 4 / 3]), gbs.GBS_E_INVAL),       # spectral: N >= 4
    ]
    for args, code in cases:
        with pytest.raises(gbs.GbsError) as e:
            gbs.gbs_create(*args, stream=0)
        assert e.value.code == code, (args, e.value)


def test_peer_neighbours_are_the_adjacent_slabs_of_the_group():
    """Host logic of gbs_bind_peers' callers: the ranks holding the slabs below / above."""
    from paper_1907_11771_b200 import gbs
    steps = list(range(2, 17, 2))
    for world, groups in ((2, 1), (4, 1), (8, 1), (8, 2), (8, 4)):
        plans = [gbs.gbs_plan("wave3d", (1024, 1024, 1024), 8, steps, world, r, groups) for r in range(world)]
        for r in range(world):
            lo, hi = gbs.peer_neighbours("wave3d", (1024, 1024, 1024), 8, steps, world, r, groups)
            me, pl, ph = plans[r], plans[lo], plans[hi]
            assert pl["my_group"] == me["my_group"] == ph["my_group"]
            s = me["slabs"]
            assert pl["my_slab"] == (me["my_slab"] - 1) % s and ph["my_slab"] == (me["my_slab"] + 1) % s
            # the lower neighbour's slab ends where this one starts (periodically)
            assert (pl["slab_z0"] + pl["slab_nz"]) % 1024 == me["slab_z0"]

"""Thin Python binding of libgbs_b200.so (include/gbs.h): argument marshalling only.

Every function has the C name and forwards to the C ABI; every step of the hot
path runs in the library's CUDA kernels.  There is no fallback: if the shared
library is missing or a CUDA device is absent the calls raise.

Device buffers are torch CUDA tensors (plumbing), host buffers numpy arrays
or CPU tensors; the stream is torch's current CUDA stream unless given.
"""

from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence

import numpy as np

from . import _build

GBS_OK = 0
GBS_E_INVAL, GBS_E_WEIGHTS, GBS_E_STATE, GBS_E_NOMEM = -1, -2, -3, -4
GBS_E_CUDA, GBS_E_NCCL, GBS_E_NONFINITE, GBS_E_UNSUPPORTED = -5, -6, -7, -8
PDE = {"adv1d": 1, "acoustic2d": 2, "wave3d": 3}
FIELDS = {"adv1d": 1, "acoustic2d": 3, "wave3d": 2}
NDIM = {"adv1d": 1, "acoustic2d": 2, "wave3d": 3}

EXPORTS = ["gbs_create", "gbs_write_state", "gbs_advance", "gbs_read_state", "gbs_write_slab",
           "gbs_read_slab", "gbs_write_slab_async", "gbs_read_slab_async", "gbs_workspace_bytes",
           "gbs_bind_workspace", "gbs_bind_peers", "gbs_sync",
           "gbs_destroy", "gbs_nccl_unique_id", "gbs_query", "gbs_plan", "gbs_halo_schedule",
           "gbs_set_option",
           "gbs_kernel_time", "gbs_strerror", "gbs_last_error", "gbs_local_hub_create",
           "gbs_local_hub_destroy", "gbs_stage_bytes", "gbs_bind_group_peers"]
GBS_TRANSPORT_NCCL, GBS_TRANSPORT_LOCAL = 0, 1


class gbs_grid(ctypes.Structure):
    _fields_ = [("pde", ctypes.c_int32), ("ndim", ctypes.c_int32),
                ("n", ctypes.c_int64 * 3), ("length", ctypes.c_double * 3)]


class gbs_dist(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int32), ("world", ctypes.c_int32), ("device", ctypes.c_int32),
                ("groups", ctypes.c_int32), ("nccl_id", ctypes.c_uint8 * 128),
                ("transport", ctypes.c_int32), ("pad", ctypes.c_int32), ("hub", ctypes.c_void_p)]


class gbs_info(ctypes.Structure):
    _fields_ = [("m", ctypes.c_int32), ("fields", ctypes.c_int32), ("radius", ctypes.c_int32),
                ("groups", ctypes.c_int32), ("slabs", ctypes.c_int32),
                ("my_group", ctypes.c_int32), ("my_slab", ctypes.c_int32),
                ("my_sequences", ctypes.c_int32), ("uses_graph", ctypes.c_int32),
                ("substeps_per_macro", ctypes.c_int64), ("my_substeps", ctypes.c_int64),
                ("slab_z0", ctypes.c_int64), ("slab_nz", ctypes.c_int64),
                ("points", ctypes.c_int64), ("macro_steps_done", ctypes.c_int64),
                ("kernel_launches", ctypes.c_int64), ("t", ctypes.c_double),
                ("bytes_per_point_substep", ctypes.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class gbs_plan_info(ctypes.Structure):
    _fields_ = [("groups", ctypes.c_int32), ("slabs", ctypes.c_int32), ("my_group", ctypes.c_int32),
                ("my_slab", ctypes.c_int32), ("my_sequences", ctypes.c_int32),
                ("my_n_k", ctypes.c_int32 * 32), ("my_substeps", ctypes.c_int64),
                ("critical_substeps", ctypes.c_int64), ("slab_z0", ctypes.c_int64),
                ("slab_nz", ctypes.c_int64)]

    def as_dict(self):
        d = {k: getattr(self, k) for k, _ in self._fields_ if k != "my_n_k"}
        d["my_n_k"] = list(self.my_n_k[: self.my_sequences])
        return d


class gbs_halo_op(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("peer", ctypes.c_int32), ("field", ctypes.c_int32),
                ("pad", ctypes.c_int32), ("plane0", ctypes.c_int64), ("planes", ctypes.c_int64)]


class GbsError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{msg} (code {code})")
        self.code = code


_lib = None


def lib_path() -> str:
    return _build.LIB


def load(build_if_missing: bool = False):
    """Load libgbs_b200.so (in-tree).  Raises if it is missing — no fallback."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_build.LIB):
        if build_if_missing:
            _build.build()
        else:
            raise ImportError(f"{_build.LIB} is missing: run `python -c 'import __graft_entry__ as g; "
                              f"g.build()'` (nvcc sm_100a) first")
    L = ctypes.CDLL(_build.LIB)
    vp, i64, dp = ctypes.c_void_p, ctypes.c_int64, ctypes.POINTER(ctypes.c_double)
    L.gbs_create.argtypes = [ctypes.POINTER(gbs_grid), ctypes.c_int, ctypes.c_int,
                             ctypes.POINTER(ctypes.c_int32), dp, ctypes.POINTER(gbs_dist), vp,
                             ctypes.POINTER(vp)]
    L.gbs_write_state.argtypes = [vp, vp, i64, ctypes.c_int]
    L.gbs_advance.argtypes = [vp, i64, ctypes.c_double]
    L.gbs_read_state.argtypes = [vp, vp, i64, ctypes.c_int]
    L.gbs_write_slab.argtypes = [vp, vp, i64, ctypes.c_int]
    L.gbs_read_slab.argtypes = [vp, vp, i64, ctypes.c_int]
    L.gbs_write_slab_async.argtypes = [vp, vp, i64, ctypes.c_int]
    L.gbs_read_slab_async.argtypes = [vp, vp, i64, ctypes.c_int]
    L.gbs_workspace_bytes.argtypes = [vp, ctypes.POINTER(ctypes.c_int64)]
    L.gbs_bind_workspace.argtypes = [vp, vp, i64]
    L.gbs_bind_peers.argtypes = [vp, vp, vp]
    L.gbs_sync.argtypes = [vp]
    L.gbs_destroy.argtypes = [vp]
    L.gbs_destroy.restype = None
    L.gbs_nccl_unique_id.argtypes = [vp]
    L.gbs_query.argtypes = [vp, ctypes.POINTER(gbs_info)]
    L.gbs_plan.argtypes = [ctypes.POINTER(gbs_grid), ctypes.c_int, ctypes.c_int,
                           ctypes.POINTER(ctypes.c_int32), ctypes.c_int, ctypes.c_int, ctypes.c_int,
                           ctypes.POINTER(gbs_plan_info)]
    L.gbs_halo_schedule.argtypes = [ctypes.c_int, ctypes.c_int, i64, ctypes.c_int, ctypes.c_uint32,
                                    ctypes.POINTER(gbs_halo_op), ctypes.c_int, ctypes.POINTER(ctypes.c_int)]
    L.gbs_set_option.argtypes = [vp, ctypes.c_char_p, i64]
    L.gbs_kernel_time.argtypes = [vp, ctypes.c_int, dp, ctypes.POINTER(i64), ctypes.c_int]
    L.gbs_stage_bytes.argtypes = [vp, ctypes.POINTER(ctypes.c_int64)]
    L.gbs_bind_group_peers.argtypes = [vp, ctypes.POINTER(vp), ctypes.POINTER(vp), ctypes.c_int]
    L.gbs_local_hub_create.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.POINTER(vp)]
    L.gbs_local_hub_destroy.argtypes = [vp]
    L.gbs_local_hub_destroy.restype = None
    L.gbs_strerror.argtypes = [ctypes.c_int]
    L.gbs_strerror.restype = ctypes.c_char_p
    L.gbs_last_error.argtypes = [vp]
    L.gbs_last_error.restype = ctypes.c_char_p
    for name in EXPORTS:
        if name not in ("gbs_destroy", "gbs_strerror", "gbs_last_error", "gbs_local_hub_destroy"):
            getattr(L, name).restype = ctypes.c_int
    _lib = L
    return L


def _check(rc: int, ctx=None):
    if rc != GBS_OK:
        L = load()
        msg = L.gbs_last_error(ctx).decode() or L.gbs_strerror(rc).decode()
        raise GbsError(rc, msg)


def _ptr_and_device(buf):
    """(address, on_device, n_values) of a torch tensor or numpy array of float64."""
    if isinstance(buf, np.ndarray):
        if buf.dtype != np.float64 or not buf.flags.c_contiguous:
            raise TypeError("host buffers must be C-contiguous float64")
        return buf.ctypes.data, 0, buf.size
    import torch
    if not isinstance(buf, torch.Tensor):
        raise TypeError("buffer must be a numpy array or a torch tensor")
    if buf.dtype != torch.float64 or not buf.is_contiguous():
        raise TypeError("tensors must be contiguous float64")
    return buf.data_ptr(), int(buf.is_cuda), buf.numel()


# ---- same names as the C ABI ------------------------------------------------
def gbs_nccl_unique_id() -> bytes:
    buf = (ctypes.c_uint8 * 128)()
    _check(load().gbs_nccl_unique_id(ctypes.cast(buf, ctypes.c_void_p)))
    return bytes(buf)


def _grid(pde: str, n: Sequence[int], length: Sequence[float] = (1.0, 1.0, 1.0)) -> gbs_grid:
    g = gbs_grid()
    g.pde = PDE[pde]
    g.ndim = NDIM[pde]
    for d in range(3):
        g.n[d] = int(n[d]) if d < len(n) else 1
        g.length[d] = float(length[d])
    return g


def gbs_plan(pde: str, n: Sequence[int], stencil_order: int, n_k: Sequence[int], world: int,
             rank: int, groups: int = 0) -> dict:
    """Host-only plan of gbs_create for (world, rank, groups): no device needed."""
    g = _grid(pde, n)
    nk = (ctypes.c_int32 * len(n_k))(*[int(x) for x in n_k])
    info = gbs_plan_info()
    _check(load().gbs_plan(ctypes.byref(g), int(stencil_order), len(n_k), nk, int(world), int(rank),
                           int(groups), ctypes.byref(info)))
    return info.as_dict()


def gbs_halo_schedule(slabs: int, my_slab: int, nz_local: int, ghost: int, field_mask: int):
    """Host-only: the ordered p2p halo operations of one slab (list of dicts)."""
    ops = (gbs_halo_op * 256)()
    n = ctypes.c_int()
    _check(load().gbs_halo_schedule(int(slabs), int(my_slab), int(nz_local), int(ghost), int(field_mask),
                                    ops, 256, ctypes.byref(n)))
    return [{"kind": "send" if o.kind == 0 else "recv", "peer": o.peer, "field": o.field,
             "plane0": o.plane0, "planes": o.planes} for o in ops[: n.value]]


def gbs_create(pde: str, n: Sequence[int], stencil_order: int, n_k: Sequence[int],
               w_k: Sequence[float], dist: Optional[dict] = None, stream=None,
               length: Sequence[float] = (1.0, 1.0, 1.0)):
    L = load()
    g = _grid(pde, n, length)
    nk = (ctypes.c_int32 * len(n_k))(*[int(x) for x in n_k])
    wk = (ctypes.c_double * len(w_k))(*[float(x) for x in w_k])
    dp = None
    if dist is not None:
        dd = gbs_dist()
        dd.rank, dd.world = int(dist["rank"]), int(dist["world"])
        dd.device, dd.groups = int(dist.get("device", 0)), int(dist.get("groups", 0))
        if dist.get("nccl_id") is not None:
            ctypes.memmove(dd.nccl_id, bytes(dist["nccl_id"]), 128)
        dd.transport = int(dist.get("transport", GBS_TRANSPORT_NCCL))
        dd.hub = dist.get("hub")
        dp = ctypes.pointer(dd)
    if stream is None:
        import torch
        stream = torch.cuda.current_stream().cuda_stream if torch.cuda.is_available() else 0
    out = ctypes.c_void_p()
    _check(L.gbs_create(ctypes.byref(g), int(stencil_order), len(n_k), nk, wk, dp,
                        ctypes.c_void_p(int(stream) if stream else 0), ctypes.byref(out)))
    return out


def gbs_local_hub_create(world: int, device: int = 0):
    """In-process transport for `world` contexts on one device (include/gbs.h)."""
    out = ctypes.c_void_p()
    _check(load().gbs_local_hub_create(int(world), int(device), ctypes.byref(out)))
    return out.value


def gbs_local_hub_destroy(hub) -> None:
    if hub:
        load().gbs_local_hub_destroy(ctypes.c_void_p(hub))


def run_local_ranks(world: int, fn, device: int = 0, groups: int = 0):
    """Run fn(dist) for rank = 0..world-1 on `world` host threads, each rank a context of this
    process on `device` joined through one local hub (GBS_TRANSPORT_LOCAL); returns the results in
    rank order and re-raises the first exception.  Test/emulation harness: the ranks share a GPU."""
    import threading
    hub = gbs_local_hub_create(world, device)
    res, err = [None] * world, [None] * world

    def body(r):
        try:
            res[r] = fn({"rank": r, "world": world, "device": device, "groups": groups,
                         "transport": GBS_TRANSPORT_LOCAL, "hub": hub})
        except BaseException as e:    # noqa: BLE001 - handed to the caller
            err[r] = e

    ts = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    gbs_local_hub_destroy(hub)
    for e in err:
        if e is not None:
            raise e
    return res


def gbs_write_state(ctx, src) -> None:
    p, dev, cnt = _ptr_and_device(src)
    _check(load().gbs_write_state(ctx, ctypes.c_void_p(p), cnt, dev), ctx)


def gbs_advance(ctx, macro_steps: int, H: float) -> None:
    _check(load().gbs_advance(ctx, int(macro_steps), float(H)), ctx)


def gbs_read_state(ctx, dst) -> None:
    p, dev, cnt = _ptr_and_device(dst)
    _check(load().gbs_read_state(ctx, ctypes.c_void_p(p), cnt, dev), ctx)


def gbs_write_slab(ctx, src) -> None:
    p, dev, cnt = _ptr_and_device(src)
    _check(load().gbs_write_slab(ctx, ctypes.c_void_p(p), cnt, dev), ctx)


def gbs_read_slab(ctx, dst) -> None:
    p, dev, cnt = _ptr_and_device(dst)
    _check(load().gbs_read_slab(ctx, ctypes.c_void_p(p), cnt, dev), ctx)


def gbs_write_slab_async(ctx, src) -> None:
    """Stage src (keep it alive and unmodified until gbs_sync) as the next state."""
    p, dev, cnt = _ptr_and_device(src)
    _check(load().gbs_write_slab_async(ctx, ctypes.c_void_p(p), cnt, dev), ctx)


def gbs_read_slab_async(ctx, dst) -> None:
    """Queue a copy of the current state into dst (complete after gbs_sync)."""
    p, dev, cnt = _ptr_and_device(dst)
    _check(load().gbs_read_slab_async(ctx, ctypes.c_void_p(p), cnt, dev), ctx)


def gbs_workspace_bytes(ctx) -> int:
    b = ctypes.c_int64(0)
    _check(load().gbs_workspace_bytes(ctx, ctypes.byref(b)), ctx)
    return b.value


def gbs_bind_peers(ctx, lower_ptr, upper_ptr) -> None:
    """Peer halo pushes (include/gbs.h): the neighbouring slabs' workspaces as device
    addresses mapped into this process (ints), or None, None to return to NCCL halos."""
    lo = ctypes.c_void_p(int(lower_ptr)) if lower_ptr else None
    hi = ctypes.c_void_p(int(upper_ptr)) if upper_ptr else None
    _check(load().gbs_bind_peers(ctx, lo, hi), ctx)


def gbs_stage_bytes(ctx) -> int:
    b = ctypes.c_int64(0)
    _check(load().gbs_stage_bytes(ctx, ctypes.byref(b)), ctx)
    return b.value


def gbs_bind_group_peers(ctx, member_workspaces, member_stages) -> None:
    """Fused combine across sequence groups: every group member's workspace and staging buffer
    as device addresses mapped into this process (ints, group order), or [] to turn it off."""
    n = len(member_workspaces)
    if n == 0:
        _check(load().gbs_bind_group_peers(ctx, None, None, 0), ctx)
        return
    W = (ctypes.c_void_p * n)(*[int(p) for p in member_workspaces])
    S = (ctypes.c_void_p * n)(*[int(p) for p in member_stages])
    _check(load().gbs_bind_group_peers(ctx, W, S, n), ctx)


def gbs_bind_workspace(ctx, ws) -> None:
    """Bind a caller-owned device buffer (a torch tensor, or None to unbind) as the state memory."""
    if ws is None:
        _check(load().gbs_bind_workspace(ctx, None, 0), ctx)
        return
    import torch
    if not (isinstance(ws, torch.Tensor) and ws.is_cuda and ws.is_contiguous()):
        raise TypeError("workspace must be a contiguous CUDA tensor")
    _check(load().gbs_bind_workspace(ctx, ctypes.c_void_p(ws.data_ptr()), ws.numel() * ws.element_size()), ctx)


def gbs_sync(ctx) -> None:
    _check(load().gbs_sync(ctx), ctx)


def gbs_destroy(ctx) -> None:
    if ctx:
        load().gbs_destroy(ctx)


def gbs_query(ctx) -> dict:
    info = gbs_info()
    _check(load().gbs_query(ctx, ctypes.byref(info)), ctx)
    return info.as_dict()


def gbs_set_option(ctx, key: str, value: int) -> None:
    _check(load().gbs_set_option(ctx, key.encode(), int(value)), ctx)


def gbs_kernel_time(ctx, cls: int, reset: bool = False):
    ms = ctypes.c_double()
    n = ctypes.c_int64()
    _check(load().gbs_kernel_time(ctx, int(cls), ctypes.byref(ms), ctypes.byref(n), int(reset)), ctx)
    return ms.value, n.value


def gbs_strerror(code: int) -> str:
    return load().gbs_strerror(int(code)).decode()


def gbs_last_error(ctx=None) -> str:
    return load().gbs_last_error(ctx).decode()


def peer_neighbours(pde, n, stencil_order, n_k, world: int, rank: int, groups: int = 0):
    """Ranks holding slab my_slab - 1 and my_slab + 1 (periodic) of this rank's sequence group,
    from the host-only plans of every rank."""
    plans = [gbs_plan(pde, n, stencil_order, n_k, world, r, groups) for r in range(world)]
    me = plans[rank]
    where = {(p["my_group"], p["my_slab"]): r for r, p in enumerate(plans)}
    return (where[(me["my_group"], (me["my_slab"] - 1) % me["slabs"])],
            where[(me["my_group"], (me["my_slab"] + 1) % me["slabs"])])


class Stepper:
    """RAII convenience around one context (still only marshalling)."""

    def __init__(self, pde, n, stencil_order, n_k, w_k, dist=None, stream=None, torch_memory=False,
                 peers=False, group_peers=False, **opts):
        self.pde = pde
        self.ctx = gbs_create(pde, n, stencil_order, n_k, w_k, dist, stream)
        for k, v in opts.items():
            gbs_set_option(self.ctx, k, v)
        self.workspace = None
        self.symm = None
        self.stage = None
        multi = bool(dist) and dist.get("world", 1) > 1 and dist.get("transport", 0) == GBS_TRANSPORT_NCCL
        if torch_memory or peers or group_peers:
            # the state buffers live in a torch tensor (PyTorch's allocator owns the memory)
            import torch
            nbytes = max(gbs_workspace_bytes(self.ctx), 1)
            if (peers or group_peers) and multi:
                self.workspace = self._peer_workspace(pde, n, stencil_order, n_k, dist, nbytes, halos=peers)
                if group_peers:
                    self._group_peers(pde, n, stencil_order, n_k, dist)
            else:
                self.workspace = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
                gbs_bind_workspace(self.ctx, self.workspace)

    def _group_peers(self, pde, n, stencil_order, n_k, dist):
        """Fused combine across GPUs (include/gbs.h gbs_bind_group_peers): a symmetric-memory
        staging buffer per rank; every member of this rank's combine (the ranks holding the same
        slab, one per sequence group) binds all members' workspaces and staging buffers."""
        import torch
        import torch.distributed as tdist
        import torch.distributed._symmetric_memory as symm
        plans = [gbs_plan(pde, n, stencil_order, n_k, dist["world"], r, dist.get("groups", 0))
                 for r in range(dist["world"])]
        me = plans[dist["rank"]]
        members = sorted((p["my_group"], r) for r, p in enumerate(plans) if p["my_slab"] == me["my_slab"])
        self.stage = symm.empty(max(gbs_stage_bytes(self.ctx), 1), dtype=torch.uint8, device="cuda")
        self.stage_symm = symm.rendezvous(self.stage, tdist.group.WORLD)
        torch.cuda.synchronize()
        tdist.barrier()
        ws_ptrs, st_ptrs = self.symm.buffer_ptrs, self.stage_symm.buffer_ptrs
        gbs_bind_group_peers(self.ctx, [ws_ptrs[r] for _, r in members], [st_ptrs[r] for _, r in members])

    def _peer_workspace(self, pde, n, stencil_order, n_k, dist, nbytes, halos=True):
        """Peer halo pushes across GPUs (include/gbs.h gbs_bind_peers): the workspace is torch
        symmetric memory, every rank's mapped into every other; the neighbours are the ranks
        holding slab my_slab -/+ 1 of the same sequence group (collective over all ranks)."""
        import torch
        import torch.distributed as tdist
        import torch.distributed._symmetric_memory as symm
        lo, hi = peer_neighbours(pde, n, stencil_order, n_k, dist["world"], dist["rank"], dist.get("groups", 0))
        ws = symm.empty(nbytes, dtype=torch.uint8, device="cuda")
        gbs_bind_workspace(self.ctx, ws)
        self.symm = symm.rendezvous(ws, tdist.group.WORLD)
        torch.cuda.synchronize()
        tdist.barrier()                          # every rank's flags are zeroed before any push
        ptrs = self.symm.buffer_ptrs
        if halos:
            gbs_bind_peers(self.ctx, ptrs[lo], ptrs[hi])
        return ws

    def write(self, y):
        gbs_write_state(self.ctx, y)

    def advance(self, macro_steps, H):
        gbs_advance(self.ctx, macro_steps, H)

    def read(self, out):
        gbs_read_state(self.ctx, out)
        return out

    def write_slab(self, y):
        gbs_write_slab(self.ctx, y)

    def read_slab(self, out):
        gbs_read_slab(self.ctx, out)
        return out

    def write_async(self, y):
        gbs_write_slab_async(self.ctx, y)

    def read_async(self, out):
        gbs_read_slab_async(self.ctx, out)
        return out

    def sync(self):
        gbs_sync(self.ctx)

    def info(self):
        return gbs_query(self.ctx)

    def close(self):
        if self.ctx:
            gbs_destroy(self.ctx)
            self.ctx = None
        self.workspace = None
        self.stage = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

#!/usr/bin/env python
"""Benchmark of the GBS hot path (BASELINE.json metric: grid-point leap-frog substeps/s and
% of HBM roofline at 1/2/4/8 B200).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5] [--impl ours|reference]
    torchrun --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N ...

One "step" = one macro step of the whole hot path (every FE / LF / final substep of every
sequence, the weighted extrapolation and, for N > 1, the cross-GPU combine) over the
workload's full grid.  Default workload: BASELINE.json configs[4] (C5, 3-D scalar wave 1024^3,
FD8, step counts {2..16}, fallback order-8 weights; the metric's 1/2/4/8-GPU config), which
fits one B200 (4 state buffers x 16 GiB).  value = grid points x S x K / max-over-ranks
device time, S = sum_k (n_k + 1) substeps per macro step.

--impl reference times the oracle (oracle/gbs_oracle.c, plain fp64 C, OpenMP over the
outer grid loop) on this host's cores on a bounded sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "grid-point leap-frog substeps/sec and % of HBM roofline at 1/2/4/8 B200"
UNIT = "grid-point-substeps/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c5")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=16)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--groups", type=int, default=0, help="sequence groups (0 = planner)")
    ap.add_argument("--opt", action="append", default=[], metavar="KEY=VALUE",
                    help="library option (gbs_set_option) for this run, e.g. pdl=0")
    ap.add_argument("--peers", action="store_true",
                    help="N > 1: halo planes pushed by the stencil kernels into the neighbours' "
                         "ghost planes through torch symmetric memory (gbs_bind_peers) instead of NCCL")
    ap.add_argument("--fused-combine", action="store_true",
                    help="N > 1 with sequence groups: the final pass stores into the owners' staging "
                         "buffers through torch symmetric memory (gbs_bind_group_peers) instead of "
                         "ncclAllReduce")
    ap.add_argument("--repeats", type=int, default=5,
                    help="extra K-step timed regions after the metric's (median / best reported "
                         "under 'repeats'; 'value' stays the first region)")
    ap.add_argument("--weights", default=None,
                    help="weight set instead of the config's (e.g. opt8: the Appendix-B optimised "
                         "weights on the config's step counts; H follows their ISB)")
    return ap.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, torch copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


class ClockSampler:
    """SM clocks and throttle reasons during the timed region (B200_PROFILING.md's clocks line):
    NVML polled every 2 ms from a thread (short regions still get samples), else
    `nvidia-smi -lms 200`."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
    BITS = [0x8, 0x40, 0x20, 0x4]              # nvmlClocksEventReason* masks, same order

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None
        self.nvml = None
        self.stop_flag = threading.Event()

    def _nvml_handle(self):
        import pynvml
        pynvml.nvmlInit()
        try:
            import torch
            uuid = str(torch.cuda.get_device_properties(self.index).uuid)
            return pynvml, pynvml.nvmlDeviceGetHandleByUUID(uuid if uuid.startswith("GPU-") else "GPU-" + uuid)
        except Exception:
            return pynvml, pynvml.nvmlDeviceGetHandleByIndex(self.index)

    def start(self):
        try:
            self.nvml = self._nvml_handle()
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
            return
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _poll(self):
        nv, h = self.nvml
        get_reasons = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            nv.nvmlDeviceGetCurrentClocksThrottleReasons
        while not self.stop_flag.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
                rs = get_reasons(h)
                mem = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_MEM)
                self.rows.append([str(sm), str(mx)] + ["Active" if rs & b else "Not Active" for b in self.BITS]
                                 + [str(mem)])
            except Exception:
                return
            self.stop_flag.wait(0.002)

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 6:
                self.rows.append(parts)

    def stop(self):
        self.stop_flag.set()
        if self.nvml:
            self.t.join(timeout=5)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        reasons = sorted({self.NAMES[i] for r in self.rows for i in range(4) if r[2 + i].lower() == "active"})
        mem = [float(r[6]) for r in self.rows if len(r) > 6 and r[6].replace(".", "").isdigit()]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "mem_mhz": statistics.median(mem) if mem else None,
                "reasons": reasons, "samples": len(self.rows), "source": "nvml" if self.nvml else "nvidia-smi"}


def workload_and_scheme(name, weights=None):
    from gbs_inputs import get_config
    from paper_1907_11771_b200 import scheme
    w = get_config(name)
    if weights:
        w = w.with_(weights=weights)
    try:
        counts, ws, _ = scheme.weight_set(w.weights, w.steps)
    except ValueError:                          # a paper scheme (e.g. GBS_8_8) brings its own counts
        counts, ws, _ = scheme.weight_set(w.weights)
    w = w.with_(steps=tuple(counts))
    wd = scheme.to_fp64(ws)
    H = scheme.macro_step(w.pde, w.order, w.n, counts, wd, w.h_factor)
    return w, counts, wd, H


def describe(w, H):
    pde = {"adv1d": "1-D advection", "acoustic2d": "2-D acoustics", "wave3d": "3-D scalar wave"}[w.pde]
    grid = "x".join(str(v) for v in w.n[: w.ndim])
    disc = "spectral" if w.order == 0 else f"FD{w.order}"
    return (f"{w.name}: {pde} {grid}, {disc}, step counts {{{','.join(map(str, w.steps))}}} "
            f"({w.weights} weights), H={H:.6g}, seeded {w.ic} IC")


# ------------------------------------------------------------------------------ oracle timing
def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.lower().startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def time_oracle_sample(w, counts, wd, H, target=1.0e9, cores=None):
    """The oracle, as it stands, on a bounded sample of workload w: one macro step on a
    grid shrunk (same PDE, stencil, scheme, H, IC recipe) to ~target pt-substeps, on
    `cores` OpenMP threads (default: every host core)."""
    import numpy as np
    from gbs_inputs import make_ic, reduced
    from oracle import c_oracle
    S = sum(n + 1 for n in counts)
    pts = max(1, int(target / S))
    if w.ndim == 3:
        e = max(16, int(round(pts ** (1 / 3) / 16)) * 16)
        n = (min(e, w.n[0]), min(e, w.n[1]), min(e, w.n[2]))
    elif w.ndim == 2:
        e = max(32, int(round(pts ** 0.5 / 32)) * 32)
        n = (min(e, w.n[0]), min(e, w.n[1]), 1)
    else:
        n = w.n
    ws = reduced(w.name, n, macro_steps=1)
    y0 = make_ic(ws)
    cores = cores or os.cpu_count() or 1
    c_oracle.set_threads(cores)
    macro = 1 if w.ndim > 1 else 20
    t0 = time.perf_counter()
    c_oracle.advance(ws.pde, ws.order, y0, counts, wd, H, macro, scale=w.n)
    dt = time.perf_counter() - t0
    units = ws.points * S * macro
    grid = "x".join(str(v) for v in n[: w.ndim])
    return {"value": units / dt, "unit": UNIT, "cores": cores, "kind": "oracle", "cpu_model": cpu_model(),
            "sample": f"{macro} macro step(s) of the {w.name} scheme (same PDE, "
                      f"{'spectral' if w.order == 0 else 'FD%d' % w.order}, steps, "
                      f"weights, H) on a {grid} grid = {units:.3g} pt-substeps in {dt:.2f} s"}


def run_reference(a):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    w, counts, wd, H = workload_and_scheme(a.config, a.weights)
    for _ in range(max(0, a.warmup)):
        time_oracle_sample(w, counts, wd, H, target=1e8)
    vals = []
    samples = []
    for _ in range(max(1, a.steps)):
        r = time_oracle_sample(w, counts, wd, H, target=2e9)
        vals.append(r["value"])
        samples.append(r)
    v = statistics.median(vals)
    cb = dict(samples[0])
    cb["value"] = v
    full_units = w.points * sum(n + 1 for n in counts)          # one macro step of the workload
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": a.gpus,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": full_units / v * 1e3,
            "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": describe(w, H), "sample": cb["sample"],
                       "ms_per_step_note": "one macro step of the full workload at the sample's measured rate"},
            "cpu_baseline": cb,
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------------ our arm
def run_ours(a):
    import torch

    from gbs_inputs import make_ic
    from paper_1907_11771_b200 import gbs

    from paper_1907_11771_b200 import dist as pdist
    rank, world, local = pdist.env()
    if world != a.gpus:
        print(f"warning: --gpus {a.gpus} but WORLD_SIZE={world}", file=sys.stderr)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        pdist.init("nccl", dev)
    w, counts, wd, H = workload_and_scheme(a.config, a.weights)
    # this rank's planes of the slowest axis (the whole grid on one GPU); every rank builds
    # only its slab of the seeded IC (bit-identical to the same planes of the full IC)
    plan = gbs.gbs_plan(w.pde, w.n, w.order, counts, world, rank, a.groups)
    srange = (plan["slab_z0"], plan["slab_z0"] + plan["slab_nz"])
    y0 = make_ic(w, srange if w.ndim > 1 else None)     # host IC (same recipe as the oracle's)
    stream = torch.cuda.Stream()
    dist_desc = None
    if world > 1:
        nccl_id = pdist.broadcast_bytes(gbs.gbs_nccl_unique_id() if rank == 0 else None, src=0)
        dist_desc = {"rank": rank, "world": world, "device": local, "groups": a.groups,
                     "nccl_id": nccl_id}

    def barrier():
        pdist.barrier(sync_cuda=True)

    def max_over_ranks(x):
        return pdist.max_over_ranks(x, dev)

    with torch.cuda.stream(stream):
        # the state buffers live in a torch tensor (gbs_bind_workspace): PyTorch owns device memory
        opts = {kv.split("=")[0]: int(kv.split("=")[1]) for kv in a.opt}
        st = gbs.Stepper(w.pde, w.n, w.order, counts, wd, dist=dist_desc, stream=stream.cuda_stream,
                         torch_memory=True, peers=a.peers and world > 1,
                         group_peers=a.fused_combine and world > 1, **opts)
        y0_dev = torch.from_numpy(y0).to("cuda", non_blocking=False)
        st.write_slab(y0_dev)
        gbs.gbs_sync(st.ctx)
        del y0_dev
        info = st.info()
        # warm-up (also builds the CUDA graph when one is used)
        st.advance(a.warmup, H)
        gbs.gbs_sync(st.ctx)
        # One step is one macro step, except on the whole-run cluster path (C1: a 2 KiB state,
        # all macro steps of a gbs_advance in one launch), where one step is the config's whole
        # run (w.macro_steps macro steps, one launch).
        whole_run = w.ndim == 1 and a.warmup >= 1 and st.info()["kernel_launches"] == 1
        # (s41: macro_steps 0 = "once around the period", ceil(1 / H) macro steps, DESIGN R22)
        run_len = (w.macro_steps if w.macro_steps > 0 else math.ceil(1.0 / H)) if whole_run else 1
        # Working sets that fit in L2 (C1, C2) are timed step by step with an L2 flush (a
        # 512 MiB write) before every timed step; larger ones run back to back.
        L2_BYTES = 126 * 2 ** 20
        flush = 6 * y0.nbytes < 2 * L2_BYTES
        scratch = torch.empty(64 * 2 ** 20, dtype=torch.float64, device=dev) if flush else None

        def timed(k):
            """k macro steps, CUDA events on the context stream; returns device ms"""
            if not flush:
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                st.advance(k * run_len, H)
                e1.record(stream)
                e1.synchronize()
                return e0.elapsed_time(e1)
            evs = []
            for _ in range(k):
                scratch.fill_(1.0)
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                st.advance(run_len, H)
                e1.record(stream)
                evs.append((e0, e1))
            evs[-1][1].synchronize()
            return sum(x.elapsed_time(y) for x, y in evs)

        # timed region 1 (the metric): K macro steps as the library runs them (CUDA-graph
        # replay), barrier + synchronize on both sides, max over ranks
        l0 = st.info()["kernel_launches"]
        clk = ClockSampler(local)
        barrier()
        clk.start()
        t_ms = timed(a.steps)
        barrier()
        clocks = pdist.merge_clocks(pdist.gather_objects(clk.stop()))
        gbs.gbs_sync(st.ctx)
        ms = max_over_ranks(t_ms)
        launches_rank = st.info()["kernel_launches"] - l0
        launches = int(pdist.sum_over_ranks(launches_rank, dev))  # the whole job's launches
        # the same region again (SURVEY §8(d) timing protocol: repeat, report median and best)
        rep_ms = [ms]
        for _ in range(max(0, a.repeats - 1)):
            barrier()
            t_r = timed(a.steps)
            barrier()
            rep_ms.append(max_over_ranks(t_r))
        # timed region 2 (the roofline): the same K macro steps with a CUDA event pair
        # recorded by the library around every stencil launch on its stream
        # (time_kernels; launched without the graph, so region 1 alone gives the metric)
        gbs.gbs_set_option(st.ctx, "time_kernels", 1)
        for cls in range(8):
            gbs.gbs_kernel_time(st.ctx, cls, reset=True)
        barrier()
        t_ms = timed(a.steps)
        barrier()
        gbs.gbs_sync(st.ctx)
        ms_instr = max_over_ranks(t_ms)
        del scratch
        ktimes = {cls: gbs.gbs_kernel_time(st.ctx, cls) for cls in range(8)}
        gbs.gbs_set_option(st.ctx, "time_kernels", 0)

    S = info["substeps_per_macro"]
    units = w.points * S * a.steps * run_len
    value = units / (ms * 1e-3)
    F = w.fields
    local_pts = w.points // max(1, info["slabs"])
    peak, peak_src = peaks()
    # kernel classes of gbs_kernel_time: (name, algorithmic bytes per point per launch)
    KCLS = {0: ("leap-frog substep", 24 * F),
            1: ("forward-Euler substep", 16 * F),
            2: ("final substep + averaging + weighted accumulate", 24 * F),
            3: ("two leap-frog substeps in one pass", 48 * F),
            4: ("leap-frog + final substep in one pass", 48 * F),
            5: ("whole-run cluster kernel", 24 * F * S * run_len),
            6: ("one single-stencil-field half of a two-substep pass", 24 * F),
            7: ("forward Euler + the first step of one leap-frog chain in one pass", 16 * F + 24 * F)}
    # bytes per point the kernel itself must read + write once (its own minimum HBM
    # traffic): the two-substep 3-D kernel moves S_u, U, S_v, P_v in and A_v, B, C_u out
    # (gbs_wave3d_pair.cuh) = 64 B instead of the metric's 2 x 24F = 96 B, and the FE
    # launch before it also writes u_2 (40 B); elsewhere it equals the metric's figure
    fused3d = w.pde == "wave3d" and (ktimes.get(3, (0, 0))[1] > 0 or ktimes.get(6, (0, 0))[1] > 0)
    # half (class 6): reads X, P and writes O1, O2 = 32 B (its 24F = 48 B algorithmic figure: each of
    # the pair's two substeps is completed by one of the two halves); LF + FIN pass: 32 B of levels
    # + 16 B accumulator in, 16 B out (FIN0: no accumulator read; counted as FINACC)
    MOVED = {0: 24 * F, 1: 16 * F + (8 if fused3d else 0), 3: 64, 4: 64, 6: 32, 7: 48}
    dom = max(ktimes, key=lambda c: ktimes[c][0])
    dom_ms, dom_n = ktimes[dom]
    avg = dom_ms / max(dom_n, 1)
    alg = KCLS[dom][1] * local_pts
    achieved = alg / (avg * 1e-3) / 1e9                                  # GB/s, algorithmic
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tr = json.load(f)
        if tr.get("config") == w.name and tr.get("class", 0) == dom:
            traffic = tr.get("lf_dram_bytes_per_launch")
    except Exception:
        pass
    others = {}
    for c, (ms_c, n_c) in ktimes.items():
        if n_c and c != dom:
            others[KCLS[c][0]] = {"avg_ms": round(ms_c / n_c, 4), "launches": n_c,
                                  "GBps_alg": round(KCLS[c][1] * local_pts / (ms_c / n_c * 1e-3) / 1e9, 1)}
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": traffic,
                "kernel": KCLS[dom][0], "algorithmic_bytes_per_launch": alg,
                "avg_launch_ms": round(avg, 4), "launches": dom_n, "peak_source": peak_src,
                "algorithmic_bytes_note": ("SURVEY.md 8(d): 24F B per point per substep x substeps per launch; "
                                           "a temporally blocked launch covers 2 substeps in one HBM pass, "
                                           "so frac can exceed 1"),
                "moved_bytes_per_launch": MOVED[dom] * local_pts if dom in MOVED else None,
                "frac_of_moved": (round(MOVED[dom] * local_pts / (avg * 1e-3) / 1e9 / peak, 4)
                                  if dom in MOVED else None),
                "share_of_step": round(dom_ms / ms_instr, 4) if ms_instr > 0 else None,
                "instrumented_ms_per_step": round(ms_instr / a.steps, 4),
                "other_kernels": others}

    # ---- end to end through the public API with host buffers (pinned), copies timed.
    # One GPU: the full-grid calls; N GPUs: each rank moves its own slab (gbs_write_slab /
    # gbs_read_slab), so no rank holds or pins the whole 16 GiB grid.
    e2e = None
    if a.e2e_steps > 0:
        # every step stages its input from pinned host memory and reads its result back;
        # the asynchronous slab IO runs those copies on the library's copy streams under
        # the neighbouring steps' macro steps; one gbs_sync at the end.  The input buffer
        # is never modified, so it is staged again each step; results alternate between
        # two host buffers (their copies are ordered on the library's d2h stream).
        with torch.cuda.stream(stream):
            h_in = torch.from_numpy(y0).pin_memory()
            h_out = [torch.empty(y0.shape, dtype=torch.float64).pin_memory() for _ in range(2)]
            # untimed: re-capture the macro-step graph (dropped when time_kernels was switched
            # off) and set up the copy streams and staging buffers
            gbs.gbs_write_slab_async(st.ctx, h_in)
            gbs.gbs_advance(st.ctx, 1, H)
            gbs.gbs_read_slab_async(st.ctx, h_out[0])
            gbs.gbs_sync(st.ctx)
            barrier()
            t0 = time.perf_counter()
            for k in range(a.e2e_steps):
                gbs.gbs_write_slab_async(st.ctx, h_in)
                gbs.gbs_advance(st.ctx, 1, H)
                gbs.gbs_read_slab_async(st.ctx, h_out[k % 2])
            gbs.gbs_sync(st.ctx)
            barrier()
            dt = max_over_ranks(time.perf_counter() - t0)
        e2e = {"value": w.points * S * a.e2e_steps / dt, "unit": UNIT, "steps": a.e2e_steps,
               "h2d_bytes_per_step": int(y0.nbytes), "d2h_bytes_per_step": int(y0.nbytes),
               "note": ("per step: gbs_write_slab_async(pinned host input) + gbs_advance(1 macro step) + "
                        "gbs_read_slab_async(pinned host result), copies on the library's copy streams "
                        "overlapping neighbouring steps; wall clock to the final gbs_sync"
                        + ("" if world == 1 else "; bytes are per rank (slab)"))}
        del h_in, h_out
    st.close()

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        cpu = time_oracle_sample(w, counts, wd, H, target=8e9)       # ~10-30 s of CPU work
        one = time_oracle_sample(w, counts, wd, H, target=5e8, cores=1)
        cpu["one_core"] = {"value": one["value"], "sample": one["sample"]}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
                "warmup": a.warmup, "ms_per_step": ms / a.steps, "higher_is_better": True,
                "macro_steps_per_step": run_len,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": describe(w, H), "grid": list(w.n[: w.ndim]), "fields": F,
                           "options": {kv.split("=")[0]: int(kv.split("=")[1]) for kv in a.opt},
                           "substeps_per_step": S * run_len,
                           "step": ("the whole %d-macro-step run in one cluster launch" % run_len if run_len > 1
                                    else "1 macro step (all sequences + combine)"),
                           "l2": ("L2 flushed (512 MiB write) before every timed macro step: working set "
                                  "%.0f MiB < 2 x L2" % (6 * y0.nbytes / 2 ** 20) if flush else
                                  "inputs larger than L2 (each state buffer %.2f GiB)" % (y0.nbytes / 2 ** 30)),
                           "plan": {"groups": info["groups"], "slabs": info["slabs"]},
                           "combine": ("none (one group)" if info["groups"] == 1 else
                                       "fused: owner ranges through symmetric memory" if a.fused_combine
                                       else "ncclAllReduce"),
                           "halo": ("peer pushes (symmetric memory)" if a.peers and world > 1 else
                                    "NCCL send/recv overlapped with the interior" if info["slabs"] > 1 else "none"),
                           "hbm_roofline_fraction_of_step": round(
                               value * 24 * F / (peak * 1e9 * world), 4),
                           # also against the nominal ~8 TB/s the north star quotes
                           "hbm_roofline_fraction_of_step_nominal_8TBps": round(
                               value * 24 * F / (8000.0 * 1e9 * world), 4)},
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
                "gpu_launches_per_rank": launches_rank,
                "sim_time_per_s": H * a.steps * run_len / (ms * 1e-3),
                "repeats": {"n": len(rep_ms),
                            "values": [round(units / (r * 1e-3), 1) for r in rep_ms],
                            "median": units / (statistics.median(rep_ms) * 1e-3),
                            "best": units / (min(rep_ms) * 1e-3)},
                "clocks": clocks}
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


def main():
    a = parse()
    if a.impl == "reference":
        return run_reference(a)
    return run_ours(a)


if __name__ == "__main__":
    sys.exit(main())

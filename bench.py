#!/usr/bin/env python3
"""Benchmark of the B200 P1 macro-face multigrid hot path.

Headline workload (BASELINE.json configs[1], "stencil-apply microbenchmark"):
the channel(16,16) mesh -- 512 macro-faces -- at refinement level 10
(268,468,225 owned DoFs), fp64. One step = one y = A x plus one r = b - A x,
each including its full ghost exchange (as the reference's apply does); the
metric is GDoF/s = 2 x owned DoFs x steps / time. Inputs x, b ~ U[-1,1]
(keyed counter RNG, seed 1, streams 0/1), resident in HBM; each vector is
2.2 GB, far larger than the 126 MB L2, so no flush is needed between steps.

Beside it, on the same run (CUDA events on the library stream, clocks sampled
through NVML during each timed region): the Jacobi and reference-GS V(2,2)
cycles on the config-2 mesh, and BASELINE configs 1, 3, 4 and 5 at their
largest size for the GPUs used (key "configs").

N > 1: one process per GPU (torchrun, or `--gpus N` alone, which re-launches
itself under torch.distributed.run); weak scaling with 512 faces per GPU
(channel(16, 16*N), reference greedy partitioner), ghost exchange over NCCL.

`--impl reference` times the reference's own CPU implementation (oracle/_ref =
the unmodified reference sources; the library is single-threaded, so one core
is all one domain can use) on the same mesh, level and step, pinned to one
host core; a 16-thread sample of independent domains is reported beside it.
"""
from __future__ import annotations

import argparse
import gc
import json
import os
import platform
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "GDoF/s for stencil apply + V(2,2) cycle (fp64) at 1/2/4/8 B200; % HBM roofline"
UNIT = "GDoF/s"
LEVEL = 10
FACES_X = 16
FACES_Y = 16


def dist_env():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(
        os.environ.get("LOCAL_RANK", "0"))


def measured_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def host_info():
    model = platform.processor() or ""
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model}


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """SM clock and throttle reasons DURING a timed region: NVML polled every
    2 ms from a thread (the library's ctypes calls release the GIL), so even a
    ~36 ms region gets samples; nvidia-smi as a fallback."""

    BITS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20, "sw_power_cap": 0x4,
            "hw_power_brake_slowdown": 0x80}

    def __init__(self, device: int):
        self.device = device
        self.sm, self.smax, self.reasons = [], 0.0, set()
        self._stop = threading.Event()
        self._nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            idx = device
            vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
            if vis:
                parts = [p.strip() for p in vis.split(",")]
                if device < len(parts) and parts[device].isdigit():
                    idx = int(parts[device])
            self._h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self._nvml = pynvml
            self.smax = float(pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM))
        except Exception:
            self._nvml = None

    def _poll(self):
        N = self._nvml
        while not self._stop.is_set():
            try:
                self.sm.append(float(N.nvmlDeviceGetClockInfo(self._h, N.NVML_CLOCK_SM)))
                bits = N.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for name, b in self.BITS.items():
                    if bits & b:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.002)

    def _smi(self):
        fields = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
                  "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                  "clocks_event_reasons.sw_power_cap")
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.device), f"--query-gpu={fields}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout
                parts = [p.strip() for p in out.strip().split(",")]
                self.sm.append(float(parts[0]))
                self.smax = max(self.smax, float(parts[1]))
                for nm, val in zip(names, parts[2:6]):
                    if val.lower().startswith("active"):
                        self.reasons.add(nm)
            except Exception:
                time.sleep(0.05)

    def __enter__(self):
        self._stop.clear()
        self.thread = threading.Thread(target=self._poll if self._nvml else self._smi, daemon=True)
        self.thread.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self.thread.join(timeout=10)

    def summary(self):
        if not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": self.smax or None, "reasons": ["unsampled"], "samples": 0,
                    "source": "nvml" if self._nvml else "nvidia-smi"}
        return {"sm_mhz": statistics.median(self.sm), "sm_max_mhz": self.smax, "reasons": sorted(self.reasons),
                "samples": len(self.sm), "source": "nvml" if self._nvml else "nvidia-smi"}


# ----------------------------------------------------------------------------- CPU reference
def _ref_cfg2_child(conn, cpu, level, steps):
    """Child process pinned to one core: the unmodified reference library on
    the config-2 mesh, apply + residual per step (the reference's apply
    includes its ghost sync)."""
    try:
        os.sched_setaffinity(0, {cpu})
        from oracle import ref as R
        mesh = R.meshgen("channel", FACES_X, FACES_Y, 1.0, 1.0)
        t0 = time.perf_counter()
        s = R.RefSession(mesh, 1, level, level, 3)
        s.fill_keyed(0, level, 1, 0)
        s.fill_keyed(1, level, 1, 1)
        setup = time.perf_counter() - t0
        dofs = s.owned(level)
        per = []
        for _ in range(steps):
            t = time.perf_counter()
            s.apply(0, 2, level)
            s.residual(1, 0, 2, level)
            per.append(time.perf_counter() - t)
        conn.send({"dofs": dofs, "step_s": per, "setup_s": setup, "cpu": cpu})
    except Exception as exc:  # pragma: no cover - reported
        conn.send({"error": repr(exc)})
    conn.close()


def cpu_reference_cfg2(level: int, steps: int):
    """(GDoF/s, seconds per step, description) of the reference on the real
    config-2 mesh, one pinned core, in a child process (so the pinning and the
    ~7 GB of reference storage do not touch the benchmark process)."""
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    a, b = ctx.Pipe(duplex=False)
    cpus = sorted(os.sched_getaffinity(0))
    cpu = cpus[-1] if cpus else 0
    p = ctx.Process(target=_ref_cfg2_child, args=(b, cpu, level, steps))
    p.start()
    out = a.recv()
    p.join()
    if "error" in out:
        raise RuntimeError(out["error"])
    secs = statistics.median(out["step_s"])
    value = 2 * out["dofs"] / secs / 1e9
    sample = (f"reference library (oracle/_ref, unmodified sources, -O3) on channel({FACES_X},{FACES_Y}) -- the "
              f"config-2 mesh, 512 faces -- at level {level} ({out['dofs']} DoFs), apply + residual per step, "
              f"{len(out['step_s'])} step(s) timed (median {secs:.2f} s; setup {out['setup_s']:.1f} s excluded), "
              f"pinned to host core {out['cpu']}")
    return value, secs, sample, len(out["step_s"])


def cpu_reference_threads(threads: int, steps: int, level: int = LEVEL):
    """All host cores: each thread owns an independent channel(2,2) sample
    domain (8 macro-faces) at the workload's level; apply + residual per step."""
    from oracle import ref as R

    mesh = R.meshgen("channel", 2, 2, 1.0, 1.0)
    sessions = []
    for t in range(threads):
        s = R.RefSession(mesh, 1, level, level, 3)
        s.fill_keyed(0, level, 1, 0)
        s.fill_keyed(1, level, 1, 1)
        sessions.append(s)
    dofs = sessions[0].owned(level)

    def work(s, k):
        for _ in range(k):
            s.apply(0, 2, level)
            s.residual(1, 0, 2, level)

    def run(k):
        ths = [threading.Thread(target=work, args=(s, k)) for s in sessions]
        t0 = time.perf_counter()
        for th in ths:
            th.start()
        for th in ths:
            th.join()
        return time.perf_counter() - t0

    run(1)
    secs = run(steps)
    value = threads * steps * 2 * dofs / secs / 1e9
    sample = (f"{threads} threads x {steps} step(s) of apply + residual, each thread an independent channel(2,2) "
              f"domain (8 faces) at level {level} ({dofs} DoFs per thread), unmodified reference library, "
              f"{secs:.1f} s")
    return value, sample


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    from oracle import ref as R
    if not R.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libhyteg_ref.so not built"}))
        return 0
    # each step (apply + residual on 268 M DoFs) takes ~20 s on one core: a bounded sample of the steps
    steps = max(1, min(args.steps, args.ref_steps))
    value, secs, sample, timed = cpu_reference_cfg2(args.level, steps)
    threads = max(1, min(os.cpu_count() or 1, 32))
    tval, tsample = cpu_reference_threads(threads, 4, args.level)
    line = {
        "metric": METRIC, "value": round(value, 5), "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "steps_timed": timed, "warmup": args.warmup, "ms_per_step": round(1e3 * secs, 1), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "cfg2: y=Ax + r=b-Ax per step (ghost sync included), P1 Laplace",
                   "mesh": f"channel({FACES_X},{FACES_Y})", "macro_faces": 512, "level": args.level,
                   "inputs": "keyed U[-1,1] seed 1, streams 0/1 (the GPU arm's values)"},
        "same_config": True,
        "impl": "reference",
        "cpu_baseline": {"value": round(value, 5), "unit": UNIT, "cores": 1, "kind": "reference", "sample": sample,
                         **host_info()},
        "all_cores_sample": {"value": round(tval, 4), "unit": UNIT, "cores": threads, "sample": tsample},
        "e2e": {"value": round(value, 5), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


# ----------------------------------------------------------------------------- GPU arm
class Ctx:
    """Per-process state shared by the benchmark legs."""

    def __init__(self, args):
        import torch.distributed as dist
        self.args = args
        self.rank, self.world, self.local = dist_env()
        self.dist = dist
        if self.world > 1 and not dist.is_initialized():
            dist.init_process_group("gloo")
        from paper_1805_10167_b200 import hytegrid as H
        self.H = H
        self.peak, self.peak_kind = measured_peak()

    def domain(self, mesh, weight_level):
        H = self.H
        if self.world > 1:
            assignment = H.partition_greedy_edgecut(mesh, self.world, weight_level)
            dom = H.DistributedDomain(mesh, self.world, assignment, local_ranks=[self.rank], device=self.local)
            uid = [H.DistributedDomain.nccl_unique_id() if self.rank == 0 else None]
            self.dist.broadcast_object_list(uid, src=0)
            dom.connect_nccl(uid[0], self.rank)
        else:
            dom = H.DistributedDomain(mesh, 1, device=self.local)
        return dom

    def barrier(self, dom):
        dom.synchronize()
        if self.world > 1:
            self.dist.barrier()

    def max_over_ranks(self, v):
        if self.world == 1:
            return v
        import torch
        t = torch.tensor([v], dtype=torch.float64)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def timed(self, dom, fn, slot=4):
        """fn() bracketed by barriers + CUDA events on the library stream, clocks
        sampled during it; returns (result, device ms max over ranks, clocks)."""
        self.barrier(dom)
        with ClockSampler(self.local) as clk:
            dom.event_record(slot)
            out = fn()
            dom.event_record(slot + 1)
            self.barrier(dom)
        return out, self.max_over_ranks(dom.event_elapsed(slot, slot + 1)), clk.summary()


def headline(c: Ctx):
    """config 2: apply + residual per step; e2e; the roofline of the residual kernel."""
    H, args = c.H, c.args
    L = args.level
    mesh = H.meshgen.channel(FACES_X, FACES_Y * c.world)
    dom = c.domain(mesh, L)
    ctl = H.Controller(dom)
    total_dofs, local_dofs = dom.owned_count(L)
    A = H.StencilOperator(dom, H.LAPLACE, L, L)
    x, b, y, r = (H.ScalarFunction(n, dom, L, L) for n in ("x", "b", "y", "r"))
    H.interpolate_random(x, L, seed=1, stream=0)
    H.interpolate_random(b, L, seed=1, stream=1)

    def step():
        H.apply(A, ctl, x, y, L)
        H.residual(A, ctl, b, x, r, L)

    for _ in range(args.warmup):
        step()
    c.barrier(dom)
    dom.profile(True)
    dom.timer_reset()
    launches0 = H.kernel_launches()
    c.barrier(dom)
    with ClockSampler(c.local) as clocks:
        dom.event_record(0)
        for _ in range(args.steps):
            step()
        dom.event_record(1)
        c.barrier(dom)
    ms = c.max_over_ranks(dom.event_elapsed(0, 1))
    launches = H.kernel_launches() - launches0
    dom.profile(False)
    res_ms, res_n = dom.timer("residual")
    app_ms, app_n = dom.timer("apply")
    value = 2.0 * total_dofs * args.steps / (ms * 1e-3) / 1e9

    # roofline of the dominant kernel: the residual launch (face interiors + edge/vertex rows as
    # trailing CTAs: every owned DoF of this rank), 24 B per DoF
    res_avg_ms = res_ms / max(res_n, 1)
    app_avg_ms = app_ms / max(app_n, 1)
    achieved = 24.0 * local_dofs / (res_avg_ms * 1e-3) / 1e9
    achieved_apply = 16.0 * local_dofs / (app_avg_ms * 1e-3) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        try:
            with open(tpath) as fh:
                traffic = json.load(fh).get(f"residual_face_L{L}")
        except Exception:
            traffic = None

    # end to end through the public API with pinned host buffers, per step: H2D of x and b,
    # apply + residual, D2H of y and r
    e2e_steps = max(1, min(args.steps, args.e2e_steps))
    hx, hb, hy, hr = (H.PinnedBuffer(local_dofs) for _ in range(4))
    x.download(L, global_order=False, out=hx.array)
    b.download(L, global_order=False, out=hb.array)
    c.barrier(dom)
    t0 = time.perf_counter()
    for _ in range(e2e_steps):  # stream-ordered: step k+1's uploads overlap step k's downloads
        x.upload_async(L, hx.array)
        b.upload_async(L, hb.array)
        step()
        y.download_async(L, hy.array)
        r.download_async(L, hr.array)
    c.barrier(dom)
    e2e_s = c.max_over_ranks(time.perf_counter() - t0)
    e2e_value = 2.0 * total_dofs * e2e_steps / e2e_s / 1e9
    del hx, hb, hy, hr

    out = {
        "value": round(value, 3), "ms_per_step": round(ms / args.steps, 4), "gpu_launches": launches,
        "clocks": clocks.summary(),
        "config": {"workload": "cfg2: y=Ax + r=b-Ax per step (ghost sync included), P1 Laplace",
                   "mesh": f"channel({FACES_X},{FACES_Y * c.world})", "macro_faces": 512 * c.world, "level": L,
                   "owned_dofs": total_dofs, "inputs": "keyed U[-1,1] seed 1, resident in HBM",
                   "l2": "inputs (2.2 GB/vector/GPU) exceed the 126 MB L2; no flush needed",
                   "parallelism": f"domain decomposition x{c.world} (greedy edge-cut), NCCL ghost exchange"},
        "roofline": {"bound": "hbm", "kernel": "k_face_stencil<RESIDUAL> (face interiors + edge/vertex rows)",
                     "achieved": round(achieved, 1), "peak": c.peak, "unit": "GB/s",
                     "frac": round(achieved / c.peak, 4), "traffic": traffic, "peak_kind": c.peak_kind,
                     "bytes_per_dof": 24, "dofs_per_launch": int(local_dofs), "avg_launch_ms": round(res_avg_ms, 4),
                     "apply_kernel": {"achieved": round(achieved_apply, 1), "frac": round(achieved_apply / c.peak, 4),
                                      "bytes_per_dof": 16, "avg_launch_ms": round(app_avg_ms, 4)}},
        "e2e": {"value": round(e2e_value, 3), "unit": UNIT, "steps": e2e_steps,
                "h2d_bytes_per_step": 2 * 8 * int(local_dofs), "d2h_bytes_per_step": 2 * 8 * int(local_dofs),
                "path": "hyb_function_upload_async (pinned H2D + scatter) -> hyb_apply + hyb_residual -> "
                        "hyb_function_download_async (gather + D2H); step k+1 uploads overlap step k downloads"},
    }
    if not args.no_vcycle:
        del x, b, y, r
        gc.collect()
        out["vcycle"] = vcycle_leg(c, dom, ctl, L, "jacobi")
        out["vcycle_gs"] = vcycle_leg(c, dom, ctl, L, "gs")
    return out


def vcycle_leg(c: Ctx, dom, ctl, L, smoother):
    """V(2,2), levels L..min on the config-2 mesh: GDoF/s per finest DoF."""
    H, args = c.H, c.args
    lmin = args.vcycle_min_level
    mg = H.GridHierarchy(dom, ctl, H.LAPLACE, lmin, L, smoother=smoother, omega=2.0 / 3.0, coarse_tol=1e-12)
    rhs = H.ScalarFunction("mg.rhs", dom, lmin, L)
    x = H.ScalarFunction("mg.x", dom, lmin, L)
    H.interpolate_random(rhs, L, seed=4, stream=0, flag_mask=H.INNER)
    for _ in range(2):
        mg.vcycle(rhs, x, L)  # warm-up (allocations, plans, graph capture)
    cycles = args.vcycles
    _, ms, clk = c.timed(dom, lambda: [mg.vcycle(rhs, x, L) for _ in range(cycles)], slot=2)
    total = dom.owned_count(L)[0]
    gdofs = total * cycles / (ms * 1e-3) / 1e9
    out = {"value": round(gdofs, 3), "unit": UNIT, "cycles": cycles, "ms_per_cycle": round(ms / cycles, 3),
           "levels": f"{L}->{lmin}", "coarse": "device CG 1e-12", "clocks": clk}
    if smoother == "jacobi":
        out["smoother"] = "weighted Jacobi 2/3, V(2,2)"
        out["roofline_frac_176B"] = round(176.0 * gdofs / c.world / c.peak, 4)
    else:
        out["smoother"] = "hybrid Gauss-Seidel (the reference GridHierarchy's smoother), V(2,2), bitwise the reference"
    return out


def cfg1_leg(c: Ctx):
    """config 1: unit square L6, 10 Jacobi V(2,2) cycles, coarse CG to 1e-14 at level 0 (one GPU: 4,225 DoFs)."""
    H = c.H
    L = 6
    mesh = H.meshgen.unit_square()
    dom = H.DistributedDomain(mesh, 1, device=c.local)
    ctl = H.Controller(dom)
    rhs, x = H.ScalarFunction("rhs", dom, 0, L), H.ScalarFunction("x", dom, 0, L)
    H.interpolate_random(rhs, L, seed=0, flag_mask=H.INNER)
    mg = H.GridHierarchy(dom, ctl, H.LAPLACE, 0, L, smoother="jacobi", coarse_tol=1e-14)
    mg.solve(rhs, x, L, 0.0, 2)
    H.interpolate(x, 0.0, L)
    rep, ms, clk = c.timed(dom, lambda: mg.solve(rhs, x, L, 0.0, 10))
    return {"mesh": "unit_square", "levels": "6->0", "dofs": dom.owned_count(L)[0], "cycles": 10,
            "ms": round(ms, 3), "ms_per_cycle": round(ms / 10, 4),
            "rate": round((rep.residuals[-1] / rep.residuals[0]) ** 0.1, 4), "clocks": clk,
            "note": "launch-latency bound (4,225 DoFs); graph-replayed cycles"}


def cfg3_leg(c: Ctx):
    """config 3: perturbed annulus 128 x 32 (8192 faces), L9, 5 V(3,3) coloured-GS cycles."""
    H = c.H
    L = c.args.cfg3_level
    mesh = H.meshgen.perturb(H.meshgen.annulus(128, 32, 1.0, 2.0), 0.1, 2)
    dom = c.domain(mesh, L)
    ctl = H.Controller(dom)
    rhs, x = H.ScalarFunction("rhs", dom, 0, L), H.ScalarFunction("x", dom, 0, L)
    H.interpolate_random(rhs, L, seed=2, flag_mask=H.INNER)
    mg = H.GridHierarchy(dom, ctl, H.LAPLACE, 0, L, smoother="colored_gs", coarse_tol=1e-12)
    for _ in range(3):  # warm-up: eager (allocations, plans), graph capture, first replay
        mg.vcycle(rhs, x, L, 3, 3)
    H.interpolate(x, 0.0, L)
    # the 5 cycles alone (the 240 B/DoF roofline is a cycle's), then the solve with its residual history
    _, ms, clk = c.timed(dom, lambda: [mg.vcycle(rhs, x, L, 3, 3) for _ in range(5)])
    mg.residual_norm(rhs, x, L)  # warm-up of the norm's path (partials buffer, first launches)
    H.interpolate(x, 0.0, L)
    rep, ms_solve, _ = c.timed(dom, lambda: mg.solve(rhs, x, L, 0.0, 5, 3, 3))
    dofs = dom.owned_count(L)[0]
    gd = dofs * 5 / (ms * 1e-3) / 1e9
    return {"mesh": "annulus(128,32) perturbed +-10% (seed 2)", "faces": 8192, "level": L, "dofs": dofs,
            "cycles": 5, "ms": round(ms, 2), "ms_per_cycle": round(ms / 5, 3), "gdof_s": round(gd, 3),
            "roofline_frac_240B": round(240.0 * gd / c.world / c.peak, 4),
            "solve_ms": round(ms_solve, 2),
            "solve_note": "solve = 5 cycles + 6 residual norms (one fused residual + r.r pass at L9 each)",
            "rate": round((rep.residuals[-1] / rep.residuals[0]) ** 0.2, 4), "clocks": clk}


def cfg4_leg(c: Ctx):
    """config 4: 64 x 64-cell square (8192 faces), FMG levels 2 -> L with Jacobi V(2,2) cycles."""
    import numpy as np
    H, args = c.H, c.args
    L = args.cfg4_level or (11 if c.world >= 8 else 10 if c.world >= 2 else 9)
    lmin = 2
    mesh = H.meshgen.channel(64, 64)
    dom = c.domain(mesh, L)
    ctl = H.Controller(dom)
    rhs, x = H.ScalarFunction("rhs", dom, lmin, L), H.ScalarFunction("x", dom, lmin, L)
    fine = H.ScalarFunction("b", dom, L, L)
    H.interpolate_random(fine, L, seed=3, lo=-1e-3, hi=1e-3, flag_mask=H.INNER)
    H.interpolate_expr(rhs, L, H.EXPR_SINSIN, [1.0, np.pi, 0.0, np.pi, 0.0, 0.0], flag_mask=H.INNER)
    H.add_scaled(rhs, 1.0, fine, L)
    H.assign(1.0, rhs, 0.0, rhs, fine, L)
    mg = H.GridHierarchy(dom, ctl, H.LAPLACE, lmin, L, smoother="jacobi", coarse_tol=args.cfg4_coarse_tol)
    mg.fmg(rhs, x, L, args.cfg4_tol, 2)  # warm: plans, graphs
    H.assign(1.0, fine, 0.0, fine, rhs, L)
    rep, ms, clk = c.timed(dom, lambda: mg.fmg(rhs, x, L, args.cfg4_tol, 60))
    dofs = dom.owned_count(L)[0]
    return {"mesh": "channel(64,64)", "faces": 8192, "levels": f"{lmin}->{L}", "dofs": dofs, "tol": args.cfg4_tol,
            "converged": rep.converged, "cycles_after_fmg": rep.iterations, "ms": round(ms, 2),
            "fmg_residual_ratio": rep.residuals[1] / rep.residuals[0],
            "final_residual_ratio": rep.residuals[-1] / rep.residuals[0], "clocks": clk,
            "note": "level 11 (137 GB per vector) needs 8 GPUs; tol 1e-7 relative is the fp64 floor of the "
                    "nodal rhs at level 9 (DESIGN.md section 7)"}


def cfg5_leg(c: Ctx):
    """config 5: 1024 faces per GPU (channel(32, 16 N)) at L11, 50 PCG iterations, V(1,1) preconditioner."""
    H, args = c.H, c.args
    L = args.cfg5_level
    mesh = H.meshgen.channel(32, 16 * c.world)
    dom = c.domain(mesh, L)
    ctl = H.Controller(dom)
    rhs, x = H.ScalarFunction("rhs", dom, L, L), H.ScalarFunction("x", dom, L, L)
    H.interpolate_random(rhs, L, seed=4, flag_mask=H.INNER)
    mg = H.GridHierarchy(dom, ctl, H.LAPLACE, 0, L, smoother="jacobi")
    mg.pcg(rhs, x, L, 3)  # warm: plans, graph capture
    rep, ms, clk = c.timed(dom, lambda: mg.pcg(rhs, x, L, 50))
    dofs = dom.owned_count(L)[0]
    gd = dofs * 50 / (ms * 1e-3) / 1e9
    return {"mesh": f"channel(32,{16 * c.world})", "faces": 1024 * c.world, "level": L, "dofs": dofs,
            "iterations": 50, "ms": round(ms, 2), "ms_per_iteration": round(ms / 50, 3), "gdof_s": round(gd, 3),
            "roofline_frac_232B": round(232.0 * gd / c.world / c.peak, 4),
            "final_residual_ratio": rep.residuals[-1] / rep.residuals[0], "clocks": clk,
            "note": "level 12 (69 GB per vector per GPU, 7 vectors) does not fit one B200: level 11 per GPU"}


def run_gpu(args):
    c = Ctx(args)
    if c.world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE {c.world}")
    if c.world > 1:  # before the library dlopens NCCL (the driver checks the ranks in the INIT lines)
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    H = c.H
    launches_all0 = H.kernel_launches()
    head = headline(c)
    gc.collect()
    configs = {}
    if not args.no_configs:
        for name in args.configs.split(","):
            if name == "cfg1" and c.world > 1:
                continue  # 4,225 DoFs: a one-GPU configuration
            try:
                configs[name] = globals()[f"{name}_leg"](c)
            except Exception as exc:  # reported, never silently dropped
                configs[name] = {"error": repr(exc)}
            gc.collect()

    cpu = None
    if c.rank == 0 and c.world == 1 and not args.no_cpu:
        try:
            cval, csecs, sample, _ = cpu_reference_cfg2(args.level, 1)
            cpu = {"value": round(cval, 5), "unit": UNIT, "cores": 1, "kind": "reference", "sample": sample,
                   **host_info()}
        except Exception as exc:  # pragma: no cover - reported, not fatal
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference", "sample": f"failed: {exc}"}

    if c.rank == 0:
        line = {
            "metric": METRIC, "value": head["value"], "unit": UNIT, "n_gpus": c.world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": head["ms_per_step"], "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": head["config"], "roofline": head["roofline"], "e2e": head["e2e"],
            "gpu_launches": head["gpu_launches"], "gpu_launches_whole_run": H.kernel_launches() - launches_all0,
            "clocks": head["clocks"], "cpu_baseline": cpu,
        }
        for k in ("vcycle", "vcycle_gs"):
            if k in head:
                line[k] = head[k]
        if configs:
            line["configs"] = configs
        print(json.dumps(line), flush=True)
    if c.world > 1:
        c.dist.barrier()
    return 0


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch_distributed(args_list, n):
    """`--gpus N` without torchrun: one process per GPU via torch.distributed.run."""
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__)] + args_list
    return subprocess.run(cmd, env=env).returncode


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--level", type=int, default=LEVEL)
    ap.add_argument("--e2e-steps", type=int, default=40)
    ap.add_argument("--ref-steps", type=int, default=2, help="timed full-mesh steps of the reference arm")
    ap.add_argument("--vcycles", type=int, default=5)
    ap.add_argument("--vcycle-min-level", type=int, default=0)
    ap.add_argument("--configs", default="cfg1,cfg3,cfg4,cfg5")
    ap.add_argument("--cfg3-level", type=int, default=9)
    ap.add_argument("--cfg4-level", type=int, default=0, help="0: 9 on 1 GPU, 10 on 2-4, 11 on 8")
    ap.add_argument("--cfg4-tol", type=float, default=1e-7)
    ap.add_argument("--cfg4-coarse-tol", type=float, default=1e-9)
    ap.add_argument("--cfg5-level", type=int, default=11)
    ap.add_argument("--no-vcycle", action="store_true")
    ap.add_argument("--no-configs", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "b200":
        print("bench.py: warmup raised to 3 (timing rules)", file=sys.stderr)
        args.warmup = 3
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return relaunch_distributed(sys.argv[1:], args.gpus)
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())

#!/usr/bin/env python3
"""Benchmark of the B200 P1 macro-face multigrid hot path.

Workload (BASELINE.json configs[1], "stencil-apply microbenchmark"): the
channel(16,16) mesh -- 512 macro-faces -- at refinement level 10
(268,468,225 owned DoFs), fp64. One step = one y = A x plus one r = b - A x,
each including its full ghost exchange (as the reference's apply does); the
metric is GDoF/s = 2 x owned DoFs x steps / time. Inputs x, b ~ U[-1,1]
(keyed counter RNG, seed 1, streams 0/1), resident in HBM; each vector is
2.2 GB, far larger than the 126 MB L2, so no flush is needed between steps.

N > 1 (torchrun, one process per GPU): weak scaling with 512 faces per GPU
(channel(16, 16*N), reference greedy partitioner), ghost exchange over NCCL.

`--impl reference` times the reference's own CPU implementation
(oracle/_ref = unmodified reference sources, single-threaded library) on the
host cores, one independent sample domain per thread.
"""
from __future__ import annotations

import argparse
import json
import os
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


class ClockSampler:
    """nvidia-smi sampling during the timed region (recipe's clocks line)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            # nvidia-smi takes a while to start: wait for its first sample so the
            # samples kept cover the timed region, then drop the pre-region ones
            t_end = time.monotonic() + 5.0
            while not self.lines and time.monotonic() < t_end and self.proc.poll() is None:
                time.sleep(0.01)
            self.lines.clear()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, smax, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = max(smax, float(parts[2]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------------------------- CPU reference
def cpu_reference_sample(threads: int, steps: int, level: int = LEVEL, warmup: int = 1):
    """The unmodified reference library (oracle/_ref) on host cores: each thread
    owns an independent sample domain channel(2,2) (8 macro-faces) at the
    workload's level and runs apply + residual (the reference's apply includes
    its ghost sync). Returns GDoF/s over all threads and a description."""
    import numpy as np

    from oracle import ref as R

    mesh = R.meshgen("channel", 2, 2, 1.0, 1.0)
    sessions = []
    for t in range(threads):
        s = R.RefSession(mesh, 1, level, level, 3)
        n = s.owned(level)
        rng = np.random.default_rng(t)
        s.set(0, level, rng.uniform(-1, 1, n))
        s.set(1, level, rng.uniform(-1, 1, n))
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

    if warmup:
        run(warmup)
    secs = run(steps)
    value = threads * steps * 2 * dofs / secs / 1e9
    sample = (f"{threads} thread(s) x {steps} step(s) of apply + residual on channel(2,2) (8 faces) at level "
              f"{level} ({dofs} DoFs per thread), unmodified reference library, {secs:.1f} s")
    return value, secs, sample


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    from oracle import ref as R
    if not R.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libhyteg_ref.so not built"}))
        return 0
    cores = os.cpu_count() or 1
    threads = max(1, min(cores, 32))
    # each step is a bounded sample: one apply + residual per thread
    value, secs, sample = cpu_reference_sample(threads, args.steps, warmup=min(args.warmup, 1))
    line = {
        "metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(1e3 * secs / args.steps, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"cfg2 apply+residual, channel({FACES_X},{FACES_Y}) shape, level {LEVEL}",
                   "sample": "channel(2,2) per thread", "level": LEVEL},
        "impl": "reference",
        "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


# ----------------------------------------------------------------------------- GPU arm
def setup_dist(world):
    import torch.distributed as dist
    if world > 1 and not dist.is_initialized():
        dist.init_process_group("gloo")
    return dist


def run_gpu(args):
    from paper_1805_10167_b200 import hytegrid as H

    rank, world, local = dist_env()
    if world > 1:
        dist = setup_dist(world)
    device = local
    L = args.level
    mesh = H.meshgen.channel(FACES_X, FACES_Y * world)
    if world > 1:
        assignment = H.partition_greedy_edgecut(mesh, world, L)
        dom = H.DistributedDomain(mesh, world, assignment, local_ranks=[rank], device=device)
        uid = [H.DistributedDomain.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        dom.connect_nccl(uid[0], rank)
    else:
        dom = H.DistributedDomain(mesh, 1, device=device)
    ctl = H.Controller(dom)
    total_dofs, local_dofs = dom.owned_count(L)
    A = H.StencilOperator(dom, H.LAPLACE, L, L)
    x = H.ScalarFunction("x", dom, L, L)
    b = H.ScalarFunction("b", dom, L, L)
    y = H.ScalarFunction("y", dom, L, L)
    r = H.ScalarFunction("r", dom, L, L)
    H.interpolate_random(x, L, seed=1, stream=0)
    H.interpolate_random(b, L, seed=1, stream=1)

    def barrier():
        dom.synchronize()
        if world > 1:
            dist.barrier()

    def step():
        H.apply(A, ctl, x, y, L)
        H.residual(A, ctl, b, x, r, L)

    for _ in range(args.warmup):
        step()
    barrier()
    dom.profile(True)
    dom.timer_reset()
    launches0 = H.kernel_launches()
    with ClockSampler(device) as clocks:
        barrier()
        dom.event_record(0)
        for _ in range(args.steps):
            step()
        dom.event_record(1)
        barrier()
    ms = dom.event_elapsed(0, 1)
    launches = H.kernel_launches() - launches0
    dom.profile(False)
    res_ms, res_n = dom.timer("residual")
    app_ms, app_n = dom.timer("apply")
    if world > 1:
        import torch
        t = torch.tensor([ms], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = 2.0 * total_dofs * args.steps / (ms * 1e-3) / 1e9

    # roofline of the dominant kernel: the residual, 24 B per DoF
    _, _, nf = H.mesh_counts(mesh)
    peak, peak_kind = measured_peak()
    res_avg_ms = res_ms / max(res_n, 1)
    app_avg_ms = app_ms / max(app_n, 1)
    # one launch covers the face interiors and, as trailing CTAs, the edge/vertex rows: every
    # owned DoF of this rank
    launch_dofs = int(local_dofs)
    achieved = 24.0 * launch_dofs / (res_avg_ms * 1e-3) / 1e9
    achieved_apply = 16.0 * launch_dofs / (app_avg_ms * 1e-3) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        try:
            with open(tpath) as fh:
                traffic = json.load(fh).get(f"residual_face_L{L}")
        except Exception:
            traffic = None

    # end to end through the public API with host buffers (pinned), per step:
    # H2D of x and b, apply + residual, D2H of y and r
    e2e_steps = max(1, min(args.steps, args.e2e_steps))
    hx = H.PinnedBuffer(local_dofs)
    hb = H.PinnedBuffer(local_dofs)
    hy = H.PinnedBuffer(local_dofs)
    hr = H.PinnedBuffer(local_dofs)
    x.download(L, global_order=False, out=hx.array)
    b.download(L, global_order=False, out=hb.array)
    barrier()
    t0 = time.perf_counter()
    # stream-ordered transfers: step k+1's uploads overlap step k's downloads
    # (full-duplex link); every step still moves its own inputs and results
    for _ in range(e2e_steps):
        x.upload_async(L, hx.array)
        b.upload_async(L, hb.array)
        step()
        y.download_async(L, hy.array)
        r.download_async(L, hr.array)
    dom.synchronize()
    barrier()
    e2e_s = time.perf_counter() - t0
    if world > 1:
        import torch
        t = torch.tensor([e2e_s], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_value = 2.0 * total_dofs * e2e_steps / e2e_s / 1e9

    # V(2,2) Jacobi cycle on the same mesh / level (levels L..2), reported beside
    vc = None
    vc_gs = None
    if not args.no_vcycle:
        vc = vcycle_bench(H, dom, ctl, L, args, world, barrier)
        vc_gs = vcycle_bench(H, dom, ctl, L, args, world, barrier, smoother="gs")

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            cores = os.cpu_count() or 1
            threads = max(1, min(cores, 32))
            cval, csecs, sample = cpu_reference_sample(threads, args.cpu_steps)
            cpu = {"value": round(cval, 4), "unit": UNIT, "cores": threads, "kind": "reference", "sample": sample}
        except Exception as exc:  # pragma: no cover - reported, not fatal
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference", "sample": f"failed: {exc}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 4), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "cfg2: y=Ax + r=b-Ax per step (ghost sync included), P1 Laplace",
                       "mesh": f"channel({FACES_X},{FACES_Y * world})", "macro_faces": nf, "level": L,
                       "owned_dofs": total_dofs, "inputs": "keyed U[-1,1] seed 1, resident in HBM",
                       "l2": "inputs (2.2 GB/vector/GPU) exceed the 126 MB L2; no flush needed",
                       "parallelism": f"domain decomposition x{world} (greedy edge-cut), NCCL ghost exchange"},
            "roofline": {"bound": "hbm", "kernel": "k_face_stencil<RESIDUAL> (face interiors + edge/vertex rows)",
                         "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 4), "traffic": traffic, "peak_kind": peak_kind,
                         "bytes_per_dof": 24, "dofs_per_launch": launch_dofs,
                         "avg_launch_ms": round(res_avg_ms, 4),
                         "apply_kernel": {"achieved": round(achieved_apply, 1), "frac": round(achieved_apply / peak, 4),
                                          "bytes_per_dof": 16, "avg_launch_ms": round(app_avg_ms, 4)}},
            "e2e": {"value": round(e2e_value, 3), "unit": UNIT, "steps": e2e_steps,
                    "h2d_bytes_per_step": 2 * 8 * local_dofs, "d2h_bytes_per_step": 2 * 8 * local_dofs,
                    "path": "hyb_function_upload_async (pinned H2D + scatter) -> hyb_apply + hyb_residual -> "
                            "hyb_function_download_async (gather + D2H); step k+1 uploads overlap step k downloads"},
            "gpu_launches": launches,
            "clocks": clocks.summary(),
            "cpu_baseline": cpu,
        }
        if vc:
            line["vcycle"] = vc
            line["vcycle_gs"] = vc_gs
        print(json.dumps(line))
    if world > 1:
        dist.barrier()
    return 0


def vcycle_bench(H, dom, ctl, L, args, world, barrier, smoother="jacobi"):
    """V(2,2), levels L..min, on the same domain: GDoF/s per finest DoF.
    smoother "jacobi" (omega 2/3; the configurations' choice) or "gs" (the
    reference GridHierarchy's own hybrid Gauss-Seidel)."""
    lmin = args.vcycle_min_level
    mg = H.GridHierarchy(dom, ctl, H.LAPLACE, lmin, L, smoother=smoother, omega=2.0 / 3.0, coarse_tol=1e-12)
    rhs = H.ScalarFunction("mg.rhs", dom, lmin, L)
    x = H.ScalarFunction("mg.x", dom, lmin, L)
    H.interpolate_random(rhs, L, seed=4, stream=0, flag_mask=H.INNER)
    mg.vcycle(rhs, x, L)  # warm-up (allocations, plans)
    barrier()
    dom.event_record(2)
    cycles = args.vcycles
    for _ in range(cycles):
        mg.vcycle(rhs, x, L)
    dom.event_record(3)
    barrier()
    ms = dom.event_elapsed(2, 3)
    if world > 1:
        import torch
        import torch.distributed as dist
        t = torch.tensor([ms], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    total = dom.owned_count(L)[0]
    peak, _ = measured_peak()
    gdofs = total * cycles / (ms * 1e-3) / 1e9
    out = {"value": round(gdofs, 3), "unit": UNIT, "cycles": cycles, "ms_per_cycle": round(ms / cycles, 3),
           "levels": f"{L}->{lmin}", "coarse": "device CG 1e-12"}
    if smoother == "jacobi":
        out["smoother"] = "weighted Jacobi 2/3, V(2,2)"
        out["roofline_frac_176B"] = round(176.0 * gdofs / world / peak, 4)
    else:
        out["smoother"] = "hybrid Gauss-Seidel (the reference GridHierarchy's smoother), V(2,2), bitwise the reference"
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--level", type=int, default=LEVEL)
    ap.add_argument("--e2e-steps", type=int, default=40)
    ap.add_argument("--cpu-steps", type=int, default=10)
    ap.add_argument("--vcycles", type=int, default=3)
    ap.add_argument("--vcycle-min-level", type=int, default=0)
    ap.add_argument("--no-vcycle", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())

"""Time BASELINE configurations 1, 3, 4 and 5 at their one-GPU sizes and print
one JSON object per configuration (device time from CUDA events on the
domain's stream; setup excluded). Configuration 2 is bench.py's headline.

  cfg1  unit square L6, 10 V(2,2) Jacobi cycles, coarse CG at level 0
  cfg3  perturbed annulus 128 x 32 (8192 faces) L9, 5 V(3,3) coloured GS
  cfg4  square 64 x 64 cells (8192 faces), FMG levels 2 -> L (default 9 on one
        GPU), V(2,2) Jacobi, cycles to tol (default 1e-7: the fp64 floor)
  cfg5  1024 faces at L11 (the per-GPU share, level 12 does not fit), 50 PCG
        iterations preconditioned by V(1,1) Jacobi
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1805_10167_b200 import hytegrid as H  # noqa: E402


def timed(dom, fn):
    dom.synchronize()
    t0 = time.perf_counter()
    dom.event_record(0)
    out = fn()
    dom.event_record(1)
    dom.synchronize()
    return out, dom.event_elapsed(0, 1), (time.perf_counter() - t0) * 1e3


def cfg1(args):
    mesh = H.meshgen.unit_square()
    L = 6
    dom = H.DistributedDomain(mesh, 1)
    ctl = H.Controller(dom)
    rhs, x = H.ScalarFunction("rhs", dom, 0, L), H.ScalarFunction("x", dom, 0, L)
    H.interpolate_random(rhs, L, seed=0, flag_mask=H.INNER)
    mg = H.GridHierarchy(dom, ctl, H.LAPLACE, 0, L, smoother="jacobi", coarse_tol=1e-14)
    mg.solve(rhs, x, L, 0.0, 2)  # warm (graph capture)
    H.interpolate(x, 0.0, L)
    rep, ms, wall = timed(dom, lambda: mg.solve(rhs, x, L, 0.0, 10))
    dofs = dom.owned_count(L)[0]
    return {"config": "cfg1", "dofs": dofs, "cycles": 10, "ms": ms, "wall_ms": wall,
            "ms_per_cycle": ms / 10, "rate": (rep.residuals[-1] / rep.residuals[0]) ** 0.1}


def cfg3(args):
    mesh = H.meshgen.perturb(H.meshgen.annulus(128, 32, 1.0, 2.0), 0.1, 2)
    L = args.cfg3_level
    dom = H.DistributedDomain(mesh, 1)
    ctl = H.Controller(dom)
    rhs, x = H.ScalarFunction("rhs", dom, 0, L), H.ScalarFunction("x", dom, 0, L)
    H.interpolate_random(rhs, L, seed=2, flag_mask=H.INNER)
    mg = H.GridHierarchy(dom, ctl, H.LAPLACE, 0, L, smoother="colored_gs", coarse_tol=1e-12)
    mg.vcycle(rhs, x, L, 3, 3)
    H.interpolate(x, 0.0, L)
    rep, ms, wall = timed(dom, lambda: mg.solve(rhs, x, L, 0.0, 5, 3, 3))
    dofs = dom.owned_count(L)[0]
    return {"config": "cfg3", "dofs": dofs, "level": L, "cycles": 5, "ms": ms, "wall_ms": wall,
            "ms_per_cycle": ms / 5, "gdof_s": dofs * 5 / ms / 1e6,
            "rate": (rep.residuals[-1] / rep.residuals[0]) ** 0.2}


def cfg4(args):
    mesh = H.meshgen.channel(64, 64)
    lmin, L = 2, args.cfg4_level
    dom = H.DistributedDomain(mesh, 1)
    ctl = H.Controller(dom)
    rhs, x = H.ScalarFunction("rhs", dom, lmin, L), H.ScalarFunction("x", dom, lmin, L)
    # sin(pi x) sin(pi y) evaluated on the device at the DoF coordinates (host numpy sin agrees to <= 4 ulp)
    H.interpolate_expr(rhs, L, H.EXPR_SINSIN, [1.0, np.pi, 0.0, np.pi, 0.0, 0.0], flag_mask=H.INNER)
    noise = H.ScalarFunction("noise", dom, L, L)
    H.interpolate_random(noise, L, seed=3, lo=-1e-3, hi=1e-3, flag_mask=H.INNER)
    H.add_scaled(rhs, 1.0, noise, L)
    del noise
    mg = H.GridHierarchy(dom, ctl, H.LAPLACE, lmin, L, smoother="jacobi", coarse_tol=args.cfg4_coarse_tol)
    fine = H.ScalarFunction("b", dom, L, L)
    H.assign(1.0, rhs, 0.0, rhs, fine, L)
    mg.fmg(rhs, x, L, args.cfg4_tol, 3)  # warm: plans, graphs
    H.assign(1.0, fine, 0.0, fine, rhs, L)
    rep, ms, wall = timed(dom, lambda: mg.fmg(rhs, x, L, args.cfg4_tol, 60))
    dofs = dom.owned_count(L)[0]
    return {"config": "cfg4", "dofs": dofs, "levels": [lmin, L], "tol": args.cfg4_tol, "converged": rep.converged,
            "cycles_after_fmg": rep.iterations, "ms": ms, "wall_ms": wall,
            "fmg_residual_ratio": rep.residuals[1] / rep.residuals[0],
            "final_residual_ratio": rep.residuals[-1] / rep.residuals[0]}


def cfg5(args):
    mesh = H.meshgen.channel(32, 16)
    L = args.cfg5_level
    dom = H.DistributedDomain(mesh, 1)
    ctl = H.Controller(dom)
    rhs, x = H.ScalarFunction("rhs", dom, L, L), H.ScalarFunction("x", dom, L, L)
    H.interpolate_random(rhs, L, seed=4, flag_mask=H.INNER)
    mg = H.GridHierarchy(dom, ctl, H.LAPLACE, 0, L, smoother="jacobi")
    mg.pcg(rhs, x, L, 3)  # warm: plans, graph capture
    rep, ms, wall = timed(dom, lambda: mg.pcg(rhs, x, L, 50))
    dofs = dom.owned_count(L)[0]
    return {"config": "cfg5", "faces": 1024, "level": L, "dofs": dofs, "iterations": 50, "ms": ms,
            "wall_ms": wall, "ms_per_iteration": ms / 50, "gdof_s": dofs * 50 / ms / 1e6,
            "final_residual_ratio": rep.residuals[-1] / rep.residuals[0]}


ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="cfg1,cfg3,cfg4,cfg5")
ap.add_argument("--cfg3-level", type=int, default=9)
ap.add_argument("--cfg4-level", type=int, default=9)
ap.add_argument("--cfg4-tol", type=float, default=1e-7)
ap.add_argument("--cfg4-coarse-tol", type=float, default=1e-9)
ap.add_argument("--cfg5-level", type=int, default=11)
args = ap.parse_args()
for name in args.configs.split(","):
    print(json.dumps(globals()[name](args)), flush=True)

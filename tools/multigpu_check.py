"""Multi-process (one process per GPU, NCCL) parity of the hot path against
a one-process run of the same mesh: the reference's P-rank model is bitwise
partition invariant (reference tests/test_solvers.cpp:464-487,
tests/test_functions.cpp:70-86), and so is this implementation, across
processes as across co-resident logical ranks.

Run under torchrun with N >= 2 GPUs (tests/test_multigpu_gpu.py does):
  python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
      tools/multigpu_check.py [--level L]
Every rank runs apply, residual, two Jacobi sweeps, one hybrid-GS sweep, one
coloured-GS sweep, restriction + prolongation, dot products, Jacobi and GS
V-cycles, FMG and PCG histories on its greedy-edge-cut share, connected over
NCCL; rank 0 gathers the owned values (keyed by global DoF index) and checks
them bitwise against its own one-process run. Prints "multigpu ok ..." and
exits 0, or raises."""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch.distributed as dist  # noqa: E402

from paper_1805_10167_b200 import hytegrid as H  # noqa: E402


def run(dom, ctl, mesh, L, owned_global):
    """the operation sequence; returns {name: owned values in global index order (local part)} and scalars"""
    out, scal = {}, {}
    A = H.StencilOperator(dom, H.LAPLACE, L - 1, L)
    x, b, y = (H.ScalarFunction(n, dom, L - 1, L) for n in ("x", "b", "y"))
    H.interpolate_random(x, L, seed=1, stream=0)
    H.interpolate_random(b, L, seed=1, stream=1)

    def grab(name, f, level=L):
        out[name] = (f.download(level, global_order=False), owned_global[level])

    H.apply(A, ctl, x, y, L)
    grab("apply", y)
    H.residual(A, ctl, b, x, y, L)
    grab("residual", y)
    scal["dot_xb"] = H.dot(x, b, L)
    scal["norm_r"] = H.norm2(y, L)
    H.smooth_jacobi(A, ctl, b, x, 2.0 / 3.0, L)
    H.smooth_jacobi(A, ctl, b, x, 2.0 / 3.0, L)
    grab("jacobi2", x)
    H.smooth_gs(A, ctl, b, x, L)
    grab("gs", x)
    H.smooth_colored_gs(A, ctl, b, x, L)
    grab("cgs", x)
    H.restrict_to_coarse(ctl, x, y, L - 1)
    grab("restrict", y, L - 1)
    H.prolongate(ctl, y, b, L - 1)
    grab("prolongate", b)
    # V-cycles (device coarse CG, NCCL allreduce of the coarse rhs), FMG, PCG
    for sm in ("jacobi", "gs"):
        mg = H.GridHierarchy(dom, ctl, H.LAPLACE, 0, L, smoother=sm)
        rhs, u = H.ScalarFunction("rhs", dom, 0, L), H.ScalarFunction("u", dom, 0, L)
        H.interpolate_random(rhs, L, seed=4, flag_mask=H.INNER)
        scal[f"vcycle_{sm}"] = tuple(mg.solve(rhs, u, L, 0.0, 4).residuals)
        grab(f"vcycle_{sm}", u)
    mg = H.GridHierarchy(dom, ctl, H.LAPLACE, 1, L, smoother="jacobi")
    rhs, u = H.ScalarFunction("rhs", dom, 1, L), H.ScalarFunction("u", dom, 1, L)
    H.interpolate_random(rhs, L, seed=3, flag_mask=H.INNER)
    scal["fmg"] = tuple(mg.fmg(rhs, u, L, 1e-8, 20).residuals)
    grab("fmg", u)
    mg = H.GridHierarchy(dom, ctl, H.LAPLACE, 0, L, smoother="jacobi")
    rhs, u = H.ScalarFunction("rhs", dom, L, L), H.ScalarFunction("u", dom, L, L)
    H.interpolate_random(rhs, L, seed=5, flag_mask=H.INNER)
    scal["pcg"] = tuple(mg.pcg(rhs, u, L, 10).residuals)
    grab("pcg", u)
    dom.synchronize()
    return out, scal


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--level", type=int, default=6)
    ap.add_argument("--mesh", default="channel", choices=["channel", "annulus"])
    args = ap.parse_args()
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    dist.init_process_group("gloo")
    L = args.level
    mesh = (H.meshgen.channel(8, 4 * world) if args.mesh == "channel"
            else H.meshgen.perturb(H.meshgen.annulus(16, 4, 1.0, 2.0), 0.1, 2))
    assignment = H.partition_greedy_edgecut(mesh, world, L)
    dom = H.DistributedDomain(mesh, world, assignment, local_ranks=[rank], device=local)
    uid = [H.DistributedDomain.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    dom.connect_nccl(uid[0], rank)
    ctl = H.Controller(dom)
    og = {lv: H.ExchangePlan(mesh, world, assignment, [rank], lv).array("owned_global") for lv in (L - 1, L)}
    mine, scal = run(dom, ctl, mesh, L, og)
    parts = [None] * world
    dist.all_gather_object(parts, (mine, scal))
    if rank == 0:
        dom1 = H.DistributedDomain(mesh, 1, device=local)
        og1 = {lv: np.arange(dom1.owned_count(lv)[0]) for lv in (L - 1, L)}
        ref, ref_scal = run(dom1, H.Controller(dom1), mesh, L, og1)
        for name, (v1, _) in ref.items():
            full = np.full(v1.size, np.nan)
            for pm, _ in parts:
                vals, gidx = pm[name]
                full[gidx] = vals
            if not np.array_equal(full, v1):
                bad = np.flatnonzero(full != v1)
                raise AssertionError(f"{name}: {bad.size} of {v1.size} differ across {world} processes")
        for name, v1 in ref_scal.items():
            for r, (_, sc) in enumerate(parts):
                if sc[name] != v1:
                    raise AssertionError(f"{name} on rank {r}: {sc[name]} vs one process {v1}")
        print(f"multigpu ok: {world} processes over NCCL, {len(ref)} fields and {len(ref_scal)} scalars/histories "
              f"bitwise equal to one process ({args.mesh}, level {L})", flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

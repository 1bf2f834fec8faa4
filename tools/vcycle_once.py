"""One warm-up + N timed Jacobi V(2,2) cycles on the config-2 mesh (for
profiling the cycle's kernel mix under ncu / timing it plainly)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1805_10167_b200 import hytegrid as H  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--level", type=int, default=10)
ap.add_argument("--min-level", type=int, default=0)
ap.add_argument("--cycles", type=int, default=1)
ap.add_argument("--smoother", default="jacobi")
ap.add_argument("--mesh", default="cfg2", help="cfg2: channel(16,16); cfg3: the perturbed annulus (8192 faces)")
ap.add_argument("--nu", type=int, nargs=2, default=(2, 2))
args = ap.parse_args()
mesh = (H.meshgen.perturb(H.meshgen.annulus(128, 32, 1.0, 2.0), 0.1, 2) if args.mesh == "cfg3"
        else H.meshgen.channel(16, 16))
dom = H.DistributedDomain(mesh, 1)
ctl = H.Controller(dom)
L = args.level
mg = H.GridHierarchy(dom, ctl, H.LAPLACE, args.min_level, L, smoother=args.smoother, omega=2.0 / 3.0, coarse_tol=1e-12)
rhs = H.ScalarFunction("rhs", dom, args.min_level, L)
x = H.ScalarFunction("x", dom, args.min_level, L)
H.interpolate_random(rhs, L, seed=4, flag_mask=H.INNER)
mg.vcycle(rhs, x, L, *args.nu)
dom.synchronize()
dom.event_record(0)
for _ in range(args.cycles):
    mg.vcycle(rhs, x, L, *args.nu)
dom.event_record(1)
ms = dom.event_elapsed(0, 1)
print(f"{ms / args.cycles:.3f} ms per cycle, residual {mg.residual_norm(rhs, x, L):.6e}")

"""Time the min-level solve of the config-4 hierarchy (square 64 x 64 cells,
level 2: 66,049 DoFs): cycles at the min level are exactly one coarse CG."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_10167_b200 import hytegrid as H  # noqa: E402

mesh = H.meshgen.channel(64, 64)
L = 2
dom = H.DistributedDomain(mesh, 1)
ctl = H.Controller(dom)
rhs, x = H.ScalarFunction("rhs", dom, L, L), H.ScalarFunction("x", dom, L, L)
H.interpolate_random(rhs, L, seed=3, flag_mask=H.INNER)
mg = H.GridHierarchy(dom, ctl, H.LAPLACE, L, L, smoother="jacobi", coarse_tol=float(sys.argv[1]) if len(sys.argv) > 1 else 1e-9)
mg.vcycle(rhs, x, L)
dom.synchronize()
dom.event_record(0)
for _ in range(5):
    H.interpolate(x, 0.0, L)
    mg.vcycle(rhs, x, L)
dom.event_record(1)
print(f"coarse solve: {dom.event_elapsed(0, 1) / 5:.3f} ms, residual {mg.residual_norm(rhs, x, L):.3e}")

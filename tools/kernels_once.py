"""Config-2 hot kernels once each (after one warm-up round): apply, residual,
Jacobi, restrict, prolongate-add, fused residual+restrict, fused prolongate-add+Jacobi at level 10 on channel(16,16) -- the command
profiled with `ncu --set full` (one launch per kernel after -s skips)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1805_10167_b200 import hytegrid as H  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 10
mesh = H.meshgen.channel(16, 16)
dom = H.DistributedDomain(mesh, 1)
ctl = H.Controller(dom)
A = H.StencilOperator(dom, H.LAPLACE, L - 1, L)
x, b, y = (H.ScalarFunction(nm, dom, L - 1, L) for nm in ("x", "b", "y"))
c = H.ScalarFunction("c", dom, L - 1, L - 1)
H.interpolate_random(x, L, seed=1, stream=0)
H.interpolate_random(b, L, seed=1, stream=1)
for _ in range(2):  # round 0 warms up, round 1 is profiled
    H.apply(A, ctl, x, y, L)
    H.residual(A, ctl, b, x, y, L)
    H.smooth_jacobi(A, ctl, b, x, 2.0 / 3.0, L)
    H.restrict_to_coarse(ctl, y, b, L - 1)
    H.prolongate_add(ctl, b, x, L - 1, H.SMOOTH_MASK)
    H.residual_restrict(A, ctl, b, x, y, c, L - 1)
    H.prolongate_add_jacobi(A, ctl, c, b, x, 2.0 / 3.0, L - 1)
dom.synchronize()
print("done")

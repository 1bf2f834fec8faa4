"""One two-sweep Jacobi pass (ST_JACOBI2) at level L on channel(16,16) after a warm-up (for ncu)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_10167_b200 import hytegrid as H  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 10
dom = H.DistributedDomain(H.meshgen.channel(16, 16), 1)
ctl = H.Controller(dom)
A = H.StencilOperator(dom, H.LAPLACE, L, L)
x, b = H.ScalarFunction("x", dom, L, L), H.ScalarFunction("b", dom, L, L)
H.interpolate_random(x, L, seed=1)
H.interpolate_random(b, L, seed=2)
for _ in range(2):
    H.smooth_jacobi2(A, ctl, b, x, 0.7, L)
dom.synchronize()
print("done")

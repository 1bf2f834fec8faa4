"""Time hybrid Gauss-Seidel sweeps vs weighted Jacobi on the config-2 mesh."""
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
for name, fn in (("gs", lambda: H.smooth_gs(A, ctl, b, x, L)), ("jacobi", lambda: H.smooth_jacobi(A, ctl, b, x, 0.7, L))):
    fn()
    dom.synchronize()
    dom.event_record(0)
    for _ in range(10):
        fn()
    dom.event_record(1)
    ms = dom.event_elapsed(0, 1) / 10
    dofs = dom.owned_count(L)[0]
    print(f"L{L} {name}: {ms:.3f} ms/sweep, {dofs / ms / 1e6:.1f} GDoF/s, {24 * dofs / ms / 1e6:.0f} GB/s algorithmic")

"""Time the fused prolongate-add + Jacobi (hyb_prolongate_add_jacobi) and a plain Jacobi sweep at
level L on the config-2 mesh, or with a second argument cfg3 on config 3's perturbed annulus (CUDA
events, after a warm-up)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_10167_b200 import hytegrid as H  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 10
which = sys.argv[2] if len(sys.argv) > 2 else "cfg2"
mesh = (H.meshgen.perturb(H.meshgen.annulus(128, 32, 1.0, 2.0), 0.1, 2) if which == "cfg3"
        else H.meshgen.channel(16, 16))
dom = H.DistributedDomain(mesh, 1)
ctl = H.Controller(dom)
A = H.StencilOperator(dom, H.LAPLACE, L - 1, L)
x, b = H.ScalarFunction("x", dom, L, L), H.ScalarFunction("b", dom, L, L)
e = H.ScalarFunction("e", dom, L - 1, L - 1)
H.interpolate_random(x, L, seed=1)
H.interpolate_random(b, L, seed=2)
H.interpolate_random(e, L - 1, seed=3, lo=-1e-3, hi=1e-3)
for name, fn in (("prolongate_add_jacobi", lambda: H.prolongate_add_jacobi(A, ctl, e, b, x, 2.0 / 3.0, L - 1)),
                 ("jacobi", lambda: H.smooth_jacobi(A, ctl, b, x, 2.0 / 3.0, L))):
    fn()
    dom.synchronize()
    dom.event_record(0)
    for _ in range(10):
        fn()
    dom.event_record(1)
    dom.synchronize()
    print(f"L{L} {name}: {dom.event_elapsed(0, 1) / 10:.3f} ms", flush=True)

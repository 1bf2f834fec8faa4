"""Config 3's mesh at one level: prolongate(add) + one coloured sweep, unfused (two calls)
and fused (hyb_prolongate_add_cgs), 10 repetitions each, CUDA events."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_10167_b200 import hytegrid as H  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 9
mesh = H.meshgen.perturb(H.meshgen.annulus(128, 32, 1.0, 2.0), 0.1, 2)
dom = H.DistributedDomain(mesh, 1)
ctl = H.Controller(dom)
A = H.StencilOperator(dom, H.LAPLACE, L - 1, L)
x, b = H.ScalarFunction("x", dom, L - 1, L), H.ScalarFunction("b", dom, L - 1, L)
e = H.ScalarFunction("e", dom, L - 1, L)
H.interpolate_random(x, L, seed=1)
H.interpolate_random(b, L, seed=2)
H.interpolate_random(e, L - 1, seed=3, lo=-1e-3, hi=1e-3)
res = []
for name, fn in (("unfused", lambda: (H.prolongate_add(ctl, e, x, L - 1, H.INNER | H.NEUMANN),
                                      H.smooth_colored_gs(A, ctl, b, x, L))),
                 ("fused", lambda: H.prolongate_add_colored_gs(A, ctl, e, b, x, L - 1))):
    fn()
    dom.synchronize()
    dom.event_record(0)
    for _ in range(10):
        fn()
    dom.event_record(1)
    dom.synchronize()
    res.append(f"{name} {dom.event_elapsed(0, 1) / 10:.3f} ms")
print(f"L{L}: " + " | ".join(res))

"""A graph-replayed Jacobi V(2,2) cycle: 5 cycles after 3 warm-ups, on config 2's channel(16,16) at
L10 -> 0 or on 8192 faces (config 3's mesh) at L9 -> 2. Usage: jac_cycles.py {cfg2|faces8192}"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_10167_b200 import hytegrid as H  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
if which == "cfg2":
    mesh, L, lmin = H.meshgen.channel(16, 16), 10, 0
else:
    mesh, L, lmin = H.meshgen.perturb(H.meshgen.annulus(128, 32, 1.0, 2.0), 0.1, 2), 9, 2
dom = H.DistributedDomain(mesh, 1)
ctl = H.Controller(dom)
mg = H.GridHierarchy(dom, ctl, H.LAPLACE, lmin, L, smoother="jacobi", coarse_tol=1e-9)
rhs, x = H.ScalarFunction("rhs", dom, lmin, L), H.ScalarFunction("x", dom, lmin, L)
H.interpolate_random(rhs, L, seed=4, flag_mask=H.INNER)
for _ in range(3):
    mg.vcycle(rhs, x, L, 2, 2)
dom.synchronize()
dom.event_record(0)
for _ in range(5):
    mg.vcycle(rhs, x, L, 2, 2)
dom.event_record(1)
dom.synchronize()
print(f"{which} L{L}->{lmin} Jacobi V(2,2): {dom.event_elapsed(0, 1) / 5:.3f} ms per cycle", flush=True)

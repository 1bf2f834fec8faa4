"""Config 3's V(3,3) coloured-GS cycle, graph-replayed: per-cycle time of 5 cycles after 3 warm-up
cycles (eager, capture, first replay). Usage: cfg3_cycles.py [level] [knob=value ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_10167_b200 import hytegrid as H  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 9
for kv in sys.argv[2:]:
    k, v = kv.split("=")
    H.tuning(k, int(v))
mesh = H.meshgen.perturb(H.meshgen.annulus(128, 32, 1.0, 2.0), 0.1, 2)
dom = H.DistributedDomain(mesh, 1)
ctl = H.Controller(dom)
mg = H.GridHierarchy(dom, ctl, H.LAPLACE, 0, L, smoother="colored_gs", coarse_tol=1e-12)
rhs, x = H.ScalarFunction("rhs", dom, 0, L), H.ScalarFunction("x", dom, 0, L)
H.interpolate_random(rhs, L, seed=4, flag_mask=H.INNER)
for _ in range(3):
    mg.vcycle(rhs, x, L, 3, 3)
dom.synchronize()
dom.event_record(0)
for _ in range(5):
    mg.vcycle(rhs, x, L, 3, 3)
dom.event_record(1)
dom.synchronize()
print(f"cfg3 L{L} {' '.join(sys.argv[2:])}: {dom.event_elapsed(0, 1) / 5:.2f} ms per cycle", flush=True)

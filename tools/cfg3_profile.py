"""Config 3 (coloured-GS V(3,3) on the perturbed annulus, L9 -> 0) with the domain's named-kernel timers
on (graphs off while profiling): where a cycle's time goes, by operation; plus the plain (graph) cycle."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_10167_b200 import hytegrid as H  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 9
if "HYB_CGS_PROLONG" in os.environ:
    H.tuning("cgs_prolong_fused", int(os.environ["HYB_CGS_PROLONG"]))
if "HYB_CGS_PAIR_MIN_N" in os.environ:
    H.tuning("cgs_pair_min_n", int(os.environ["HYB_CGS_PAIR_MIN_N"]))
cyc = 3
mesh = H.meshgen.perturb(H.meshgen.annulus(128, 32, 1.0, 2.0), 0.1, 2)
dom = H.DistributedDomain(mesh, 1)
ctl = H.Controller(dom)
mg = H.GridHierarchy(dom, ctl, H.LAPLACE, 0, L, smoother="colored_gs", coarse_tol=1e-12)
rhs, x = H.ScalarFunction("rhs", dom, 0, L), H.ScalarFunction("x", dom, 0, L)
H.interpolate_random(rhs, L, seed=4, flag_mask=H.INNER)
mg.vcycle(rhs, x, L, 3, 3)
dom.synchronize()
dom.event_record(0)
for _ in range(cyc):
    mg.vcycle(rhs, x, L, 3, 3)
dom.event_record(1)
dom.synchronize()
print(f"plain: {dom.event_elapsed(0, 1) / cyc:.2f} ms per cycle")
dom.profile(True)
dom.timer_reset()
dom.event_record(0)
for _ in range(cyc):
    mg.vcycle(rhs, x, L, 3, 3)
dom.event_record(1)
dom.synchronize()
tot = dom.event_elapsed(0, 1) / cyc
print(f"profiled: {tot:.2f} ms per cycle")
acc = 0.0
for name in ("coloured_gs_pair", "coloured_gs_prolong", "coloured_gs", "residual_restrict", "restrict", "prolongate_add", "prolongate", "coarse_cg", "apply"):
    ms, n = dom.timer(name)
    if n:
        acc += ms / cyc
        print(f"  {name:20s} {ms / cyc:8.2f} ms  {n // cyc:5d} launches per cycle")
print(f"  {'other (syncs, edges)':20s} {tot - acc:8.2f} ms")

"""Config 4 (FMG on channel(64,64), levels 2->9) with the domain's named-kernel
timers on (CUDA events around each hot launch; graphs off while profiling):
where the FMG solve's time goes, by operation."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_10167_b200 import hytegrid as H  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 9
mesh = H.meshgen.channel(64, 64)
dom = H.DistributedDomain(mesh, 1)
ctl = H.Controller(dom)
rhs, x = H.ScalarFunction("rhs", dom, 2, L), H.ScalarFunction("x", dom, 2, L)
H.interpolate_expr(rhs, L, H.EXPR_SINSIN, [1.0, np.pi, 0.0, np.pi, 0.0, 0.0], flag_mask=H.INNER)
mg = H.GridHierarchy(dom, ctl, H.LAPLACE, 2, L, smoother="jacobi", coarse_tol=1e-9)
fine = H.ScalarFunction("b", dom, L, L)
H.assign(1.0, rhs, 0.0, rhs, fine, L)
mg.fmg(rhs, x, L, 1e-7, 3)
H.assign(1.0, fine, 0.0, fine, rhs, L)
H.interpolate(x, 0.0, L)
dom.synchronize()
dom.profile(True)
dom.timer_reset()
dom.event_record(0)
rep = mg.fmg(rhs, x, L, 1e-7, 60)
dom.event_record(1)
dom.synchronize()
total = dom.event_elapsed(0, 1)
print(f"fmg total {total:.1f} ms (profiled, graphs off), cycles after fmg {rep.iterations}")
for name in ("coarse_cg", "jacobi", "jacobi_zero", "residual", "residual_restrict", "prolongate_jacobi", "prolongate",
             "prolongate_add", "restrict", "apply"):
    ms, n = dom.timer(name)
    if n:
        print(f"  {name:20s} {ms:8.2f} ms  {n:5d} launches")

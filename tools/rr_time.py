"""Time the fused residual + restriction (fine level L -> L-1) on config 3's perturbed annulus (8192
faces) or config 2's channel(16,16): whole operation and its face kernel (the domain's named timer).
Usage: rr_time.py {cfg3|cfg2} L [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_10167_b200 import hytegrid as H  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
L = int(sys.argv[2]) if len(sys.argv) > 2 else 9
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
mesh = (H.meshgen.perturb(H.meshgen.annulus(128, 32, 1.0, 2.0), 0.1, 2) if which == "cfg3"
        else H.meshgen.channel(16, 16))
dom = H.DistributedDomain(mesh, 1)
ctl = H.Controller(dom)
A = H.StencilOperator(dom, H.LAPLACE, L - 1, L)
x, b, r = (H.ScalarFunction(n, dom, L, L) for n in ("x", "b", "r"))
c = H.ScalarFunction("c", dom, L - 1, L - 1)
H.interpolate_random(x, L, seed=1)
H.interpolate_random(b, L, seed=2)
H.residual_restrict(A, ctl, b, x, r, c, L - 1)
dom.synchronize()
dom.profile(True)
dom.timer_reset()
dom.event_record(0)
for _ in range(reps):
    H.residual_restrict(A, ctl, b, x, r, c, L - 1)
dom.event_record(1)
dom.synchronize()
tot = dom.event_elapsed(0, 1) / reps
ms, n = dom.timer("residual_restrict")
dofs = dom.owned_count(L)[0]
print(f"{which} L{L} residual_restrict: {tot:.3f} ms per call (face kernel {ms / max(n, 1):.3f} ms = "
      f"{18.0 * dofs / (ms / max(n, 1)) * 1e-6:.0f} GB/s at 18 B/DoF)", flush=True)

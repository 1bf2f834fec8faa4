"""Config 3's mesh at one level: 10 coloured sweeps as 10 single sweeps and as 5 pairs
(hyb_smooth_cgs_n), CUDA events around each, plus the face kernels' own timers."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_10167_b200 import hytegrid as H  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 9
mesh = H.meshgen.perturb(H.meshgen.annulus(128, 32, 1.0, 2.0), 0.1, 2)
dom = H.DistributedDomain(mesh, 1)
ctl = H.Controller(dom)
A = H.StencilOperator(dom, H.LAPLACE, L, L)
x, b = H.ScalarFunction("x", dom, L, L), H.ScalarFunction("b", dom, L, L)
H.interpolate_random(x, L, seed=1)
H.interpolate_random(b, L, seed=2)
H.tuning("cgs_pair_min_n", 256)
for name, fn in (("single x10", lambda: [H.smooth_colored_gs(A, ctl, b, x, L) for _ in range(10)]),
                 ("pair x5", lambda: H.smooth_colored_gs(A, ctl, b, x, L, count=10))):
    fn()
    dom.synchronize()
    dom.event_record(0)
    fn()
    dom.event_record(1)
    dom.synchronize()
    plain = dom.event_elapsed(0, 1)
    dom.profile(True)
    dom.timer_reset()
    fn()
    dom.synchronize()
    k = [f"{t} {dom.timer(t)[0] / max(dom.timer(t)[1], 1):.3f} ms x{dom.timer(t)[1]}"
         for t in ("coloured_gs", "coloured_gs_pair") if dom.timer(t)[1]]
    dom.profile(False)
    print(f"L{L} {name}: {plain / 10:.3f} ms per sweep | " + " | ".join(k))

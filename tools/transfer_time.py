"""Time restrict_to_coarse and prolongate_add (coarse level L-1 -> L) on a mesh:
config 3's perturbed annulus (8192 faces) or config 2's channel(16,16).
Usage: transfer_time.py {cfg3|cfg2} L"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_10167_b200 import hytegrid as H  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
L = int(sys.argv[2]) if len(sys.argv) > 2 else 9
mesh = (H.meshgen.perturb(H.meshgen.annulus(128, 32, 1.0, 2.0), 0.1, 2) if which == "cfg3"
        else H.meshgen.channel(16, 16))
dom = H.DistributedDomain(mesh, 1)
ctl = H.Controller(dom)
f = H.ScalarFunction("f", dom, L, L)
c = H.ScalarFunction("c", dom, L - 1, L - 1)
H.interpolate_random(f, L, seed=1)
H.interpolate_random(c, L - 1, seed=2)
for name, fn in (("restrict", lambda: H.restrict_to_coarse(ctl, f, c, L - 1)),
                 ("prolongate_add", lambda: H.prolongate_add(ctl, c, f, L - 1, H.SMOOTH_MASK))):
    fn()
    dom.synchronize()
    dom.event_record(0)
    for _ in range(10):
        fn()
    dom.event_record(1)
    dom.synchronize()
    print(f"{which} L{L} {name}: {dom.event_elapsed(0, 1) / 10:.3f} ms", flush=True)

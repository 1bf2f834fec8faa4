"""V-cycle (config 2, L10 -> 0) and config-1 cycle times with the coarse-end kernel off / on, for a
given dofs-per-CTA setting (HYB_MEGA_DPC)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_10167_b200 import hytegrid as H  # noqa: E402
H.tuning("mega_dofs_per_cta", int(os.environ.get("HYB_MEGA_DPC", "16384")))
res = []
for mesh, L, cyc in ((H.meshgen.channel(16, 16), 10, 10), (H.meshgen.unit_square(), 6, 50)):
    for mega in (False, True):
        dom = H.DistributedDomain(mesh, 1)
        ctl = H.Controller(dom)
        mg = H.GridHierarchy(dom, ctl, H.LAPLACE, 0, L, smoother="jacobi", coarse_tol=1e-12)
        mg.use_mega(mega, int(os.environ.get("HYB_MEGA_MAXN", "64")))
        rhs, x = H.ScalarFunction("b", dom, 0, L), H.ScalarFunction("x", dom, 0, L)
        H.interpolate_random(rhs, L, seed=4, flag_mask=H.INNER)
        for _ in range(3):
            mg.vcycle(rhs, x, L, 2, 2)
        dom.synchronize()
        dom.event_record(0)
        for _ in range(cyc):
            mg.vcycle(rhs, x, L, 2, 2)
        dom.event_record(1)
        dom.synchronize()
        res.append(f"L{L} mega={int(mega)} {dom.event_elapsed(0, 1) / cyc:.3f} ms")
print(" | ".join(res))

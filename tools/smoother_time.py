"""Time one smoother sweep at a configuration's finest level (CUDA events on
the domain stream, after a warm-up sweep) -- the command profiled with ncu for
the smoother kernels:
  cgs  coloured GS on config 3's perturbed annulus (8192 faces), L9
  gs   the reference's hybrid GS on config 2's channel(16,16), L10
  jac  weighted Jacobi on the same mesh as the smoother it is compared with
Usage: smoother_time.py {cgs|gs} [level] [sweeps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_10167_b200 import hytegrid as H  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "cgs"
if which == "cgs":
    mesh, L = H.meshgen.perturb(H.meshgen.annulus(128, 32, 1.0, 2.0), 0.1, 2), 9
else:
    mesh, L = H.meshgen.channel(16, 16), 10
L = int(sys.argv[2]) if len(sys.argv) > 2 else L
sweeps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
dom = H.DistributedDomain(mesh, 1)
ctl = H.Controller(dom)
A = H.StencilOperator(dom, H.LAPLACE, L, L)
x, b = H.ScalarFunction("x", dom, L, L), H.ScalarFunction("b", dom, L, L)
H.interpolate_random(x, L, seed=1)
H.interpolate_random(b, L, seed=2)
smooth = {"cgs": lambda: H.smooth_colored_gs(A, ctl, b, x, L),
          "gs": lambda: H.smooth_gs(A, ctl, b, x, L)}[which]
dofs = dom.owned_count(L)[0]
timer = {"cgs": "coloured_gs", "gs": "gauss_seidel", "jacobi": "jacobi"}
for name, fn in ((which, smooth), ("jacobi", lambda: H.smooth_jacobi(A, ctl, b, x, 2.0 / 3.0, L))):
    fn()
    dom.synchronize()
    dom.profile(True)
    dom.timer_reset()
    dom.event_record(0)
    for _ in range(sweeps):
        fn()
    dom.event_record(1)
    dom.synchronize()
    dom.profile(False)
    ms = dom.event_elapsed(0, 1) / sweeps
    kms, kn = dom.timer(timer[name])
    kms /= max(kn, 1)
    print(f"L{L} {name}: {ms:.3f} ms/sweep (face kernel {kms:.3f} ms = {24 * dofs / kms / 1e6:.0f} GB/s), "
          f"{dofs / ms / 1e6:.1f} GDoF/s, {24 * dofs / ms / 1e6:.0f} GB/s algorithmic (24 B/DoF)", flush=True)

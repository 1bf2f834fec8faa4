import sys
import numpy as np
sys.path.insert(0, ".")
from paper_1805_10167_b200 import hytegrid as H
from tests.helpers import keyed_uniform
mesh = H.meshgen.unit_square()
for L, bc in ((7, None), (8, None), (8, {1: H.NEUMANN})):
    outs = []
    for mega in (False, True):
        dom = H.DistributedDomain(mesh, 1)
        ctl = H.Controller(dom)
        mg = H.GridHierarchy(dom, ctl, H.LAPLACE, 0, L, bc=bc, smoother="jacobi", coarse_tol=1e-12)
        mg.use_mega(mega)
        mg.use_graphs(False)
        rhs, x = H.ScalarFunction("b", dom, 0, L, bc), H.ScalarFunction("x", dom, 0, L, bc)
        rhs.upload(L, keyed_uniform(mesh, L, 9))
        try:
            mg.vcycle(rhs, x, L, 2, 2)
            outs.append(x.download(L))
        except Exception as e:
            outs.append(None)
            print(L, bc, mega, "ERR", str(e)[:160])
    if all(o is not None for o in outs):
        d = np.abs(outs[0] - outs[1])
        print(L, bc, "maxdiff", d.max(), "ndiff", np.count_nonzero(d), "of", d.size)

"""GridHierarchy.residual_norm takes r.r from the residual kernel's own CTAs (residual_dot): the value must
agree with the composed residual + dot (reference src/solvers.cpp:444-449) to rounding, leave the same r
behind bitwise, and be bitwise invariant under the partition (fixed partial shapes), as dot is."""
import numpy as np
import pytest

from paper_1805_10167_b200 import hytegrid as H
from tests.helpers import FIXTURES, keyed_uniform

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("mesh_name,L", [("square", 6), ("ring8", 5), ("channel21", 9)])
def test_residual_norm_matches_residual_plus_dot(mesh_name, L):
    mesh = FIXTURES[mesh_name]()
    norms = []
    for ranks in (1, 2, 3):
        dom = H.DistributedDomain(mesh, ranks)
        ctl = H.Controller(dom)
        A = H.StencilOperator(dom, H.LAPLACE, 0, L)
        rhs, x, r = (H.ScalarFunction(n, dom, 0, L) for n in ("rhs", "x", "r"))
        rhs.upload(L, keyed_uniform(mesh, L, seed=91))
        x.upload(L, keyed_uniform(mesh, L, seed=92))
        mg = H.GridHierarchy(dom, ctl, H.LAPLACE, 0, L, smoother="jacobi")
        got = mg.residual_norm(rhs, x, L)
        H.residual(A, ctl, rhs, x, r, L)
        want = np.sqrt(H.dot(r, r, L))
        assert abs(got - want) <= 1e-13 * want, (mesh_name, ranks, got, want)
        norms.append(got)
    assert norms[0] == norms[1] == norms[2], norms

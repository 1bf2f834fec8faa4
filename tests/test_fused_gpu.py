"""GPU: the V-cycle's fused residual + restriction (hyb_residual_restrict)
equals residual followed by restrict_to_coarse, bitwise, on every owned
coarse DoF (the composed pair is itself bitwise the reference's, see
test_parity_gpu.py)."""
import numpy as np
import pytest

from paper_1805_10167_b200 import hytegrid as H
from tests.helpers import FIXTURES, keyed_uniform

pytestmark = pytest.mark.gpu

BCS = {"dirichlet": None, "mixed": {1: H.DIRICHLET, 2: H.NEUMANN}}


@pytest.mark.parametrize("mesh_name", ["square", "square_rev", "ring8", "channel21", "tri"])
@pytest.mark.parametrize("ranks", [1, 3])
@pytest.mark.parametrize("bc", ["dirichlet", "mixed"])
def test_residual_restrict_bitwise(mesh_name, ranks, bc):
    mesh = FIXTURES[mesh_name]()
    bcd = BCS[bc]
    for L in (1, 2, 3, 5, 7):
        dom = H.DistributedDomain(mesh, ranks)
        ctl = H.Controller(dom)
        A = H.StencilOperator(dom, H.LAPLACE, L, L, bcd)
        rhs = H.ScalarFunction("rhs", dom, L, L, bcd)
        x = H.ScalarFunction("x", dom, L, L, bcd)
        r = H.ScalarFunction("r", dom, L, L, bcd)
        c1 = H.ScalarFunction("c1", dom, L - 1, L - 1, bcd)
        c2 = H.ScalarFunction("c2", dom, L - 1, L - 1, bcd)
        rhs.upload(L, keyed_uniform(mesh, L, seed=71))
        x.upload(L, keyed_uniform(mesh, L, seed=72))
        H.residual(A, ctl, rhs, x, r, L)
        H.restrict_to_coarse(ctl, r, c1, L - 1)
        r2 = H.ScalarFunction("r2", dom, L, L, bcd)
        H.residual_restrict(A, ctl, rhs, x, r2, c2, L - 1)
        assert np.array_equal(c1.download(L - 1), c2.download(L - 1)), (mesh_name, ranks, bc, L)


def test_residual_restrict_cfg2_shape_level9():
    """512 faces, fine level 9: every band/column-block boundary of the fused kernel."""
    mesh = H.meshgen.channel(16, 16)
    L = 9
    dom = H.DistributedDomain(mesh, 1)
    ctl = H.Controller(dom)
    A = H.StencilOperator(dom, H.LAPLACE, L, L)
    rhs, x, r = (H.ScalarFunction(n, dom, L, L) for n in ("rhs", "x", "r"))
    c1, c2 = (H.ScalarFunction(n, dom, L - 1, L - 1) for n in ("c1", "c2"))
    H.interpolate_random(rhs, L, seed=73)
    H.interpolate_random(x, L, seed=74)
    H.residual(A, ctl, rhs, x, r, L)
    H.restrict_to_coarse(ctl, r, c1, L - 1)
    H.residual_restrict(A, ctl, rhs, x, r, c2, L - 1)
    assert np.array_equal(c1.download(L - 1), c2.download(L - 1))


def test_residual_restrict_argument_checks():
    mesh = FIXTURES["square"]()
    dom = H.DistributedDomain(mesh, 1)
    ctl = H.Controller(dom)
    A = H.StencilOperator(dom, H.LAPLACE, 3, 3)
    f = H.ScalarFunction("f", dom, 2, 3)
    g = H.ScalarFunction("g", dom, 2, 3)
    with pytest.raises(H.InvalidArgument):
        H.residual_restrict(A, ctl, f, g, g, f, 2)
    with pytest.raises(H.OutOfRange):
        H.residual_restrict(A, ctl, f, g, H.ScalarFunction("r", dom, 3, 3), f, 3)


@pytest.mark.parametrize("mesh_name", ["square", "square_rev", "ring8", "channel21", "tri"])
@pytest.mark.parametrize("ranks", [1, 3])
@pytest.mark.parametrize("bc", ["dirichlet", "mixed"])
def test_prolongate_add_jacobi_bitwise(mesh_name, ranks, bc):
    """The cycle's correction + first post-smoothing sweep, fused, equals
    prolongate_add then smooth_jacobi bitwise on every owned DoF."""
    mesh = FIXTURES[mesh_name]()
    bcd = BCS[bc]
    for L in (1, 2, 3, 4, 5, 7):
        out = []
        for fused in (False, True):
            dom = H.DistributedDomain(mesh, ranks)
            ctl = H.Controller(dom)
            A = H.StencilOperator(dom, H.LAPLACE, L, L, bcd)
            rhs = H.ScalarFunction("rhs", dom, L, L, bcd)
            x = H.ScalarFunction("x", dom, L, L, bcd)
            e = H.ScalarFunction("e", dom, L - 1, L - 1, bcd)
            rhs.upload(L, keyed_uniform(mesh, L, seed=81))
            x.upload(L, keyed_uniform(mesh, L, seed=82))
            e.upload(L - 1, keyed_uniform(mesh, L - 1, seed=83))
            if fused:
                H.prolongate_add_jacobi(A, ctl, e, rhs, x, 0.7, L - 1)
            else:
                H.prolongate_add(ctl, e, x, L - 1, H.SMOOTH_MASK)
                H.smooth_jacobi(A, ctl, rhs, x, 0.7, L)
            out.append(x.download(L))
        assert np.array_equal(out[0], out[1]), (mesh_name, ranks, bc, L)


def test_prolongate_add_jacobi_cfg2_shape_level9():
    """512 faces, fine level 9: band and column-block boundaries of the fused kernel."""
    mesh = H.meshgen.channel(16, 16)
    L = 9
    out = []
    for fused in (False, True):
        dom = H.DistributedDomain(mesh, 1)
        ctl = H.Controller(dom)
        A = H.StencilOperator(dom, H.LAPLACE, L, L)
        rhs, x = H.ScalarFunction("rhs", dom, L, L), H.ScalarFunction("x", dom, L, L)
        e = H.ScalarFunction("e", dom, L - 1, L - 1)
        H.interpolate_random(rhs, L, seed=84)
        H.interpolate_random(x, L, seed=85)
        H.interpolate_random(e, L - 1, seed=86)
        if fused:
            H.prolongate_add_jacobi(A, ctl, e, rhs, x, 2.0 / 3.0, L - 1)
        else:
            H.prolongate_add(ctl, e, x, L - 1, H.SMOOTH_MASK)
            H.smooth_jacobi(A, ctl, rhs, x, 2.0 / 3.0, L)
        out.append(x.download(L))
    assert np.array_equal(out[0], out[1])

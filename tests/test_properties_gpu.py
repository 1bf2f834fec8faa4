"""GPU: the reference's structural tests of the transfer operators and the
smoothers (tests/test_solvers.cpp:158-270, tests/test_operators.cpp:287-351,
tests/test_solvers.cpp:394-406), run on the device path.
"""
import numpy as np
import pytest

from paper_1805_10167_b200 import hytegrid as H
from tests.helpers import FIXTURES, keyed_uniform

pytestmark = pytest.mark.gpu

MESHES = ["square", "square_rev", "ring8", "channel21", "tri"]


@pytest.mark.parametrize("mesh_name", MESHES)
@pytest.mark.parametrize("ranks", [1, 2])
def test_prolongation_reproduces_linear_functions(mesh_name, ranks):
    """P of a linear function is the linear function (tests/test_solvers.cpp:158-174)."""
    mesh = FIXTURES[mesh_name]()
    dom = H.DistributedDomain(mesh, ranks)
    ctl = H.Controller(dom)
    f = H.ScalarFunction("f", dom, 3, 4)
    lin = lambda x, y: 0.25 - 1.5 * x + 2.0 * y  # noqa: E731
    H.interpolate(f, lin, 3)
    H.prolongate(ctl, f, f, 3)
    xy = dom.coords(4)
    want = lin(xy[:, 0], xy[:, 1])
    assert np.max(np.abs(f.download(4) - want)) <= 1e-13


@pytest.mark.parametrize("mesh_name", MESHES)
@pytest.mark.parametrize("ranks", [1, 3])
def test_restriction_is_the_transpose_of_prolongation(mesh_name, ranks):
    """(R u, v)_coarse == (u, P v)_fine on all DoFs (tests/test_solvers.cpp:201-229)."""
    mesh = FIXTURES[mesh_name]()
    L = 4
    dom = H.DistributedDomain(mesh, ranks)
    ctl = H.Controller(dom)
    u = H.ScalarFunction("u", dom, L, L)
    Ru = H.ScalarFunction("Ru", dom, L - 1, L - 1)
    v = H.ScalarFunction("v", dom, L - 1, L - 1)
    Pv = H.ScalarFunction("Pv", dom, L, L)
    u.upload(L, keyed_uniform(mesh, L, seed=5))
    v.upload(L - 1, keyed_uniform(mesh, L - 1, seed=6))
    H.restrict_to_coarse(ctl, u, Ru, L - 1)
    H.prolongate(ctl, v, Pv, L - 1)
    a = H.dot(Ru, v, L - 1)
    b = H.dot(u, Pv, L)
    assert abs(a - b) <= 1e-13 * (abs(a) + abs(b) + 1.0), (a, b)


@pytest.mark.parametrize("mesh_name", MESHES)
@pytest.mark.parametrize("form", [H.LAPLACE, H.MASS])
def test_galerkin_coarse_operator(mesh_name, form):
    """A_c v == R (A (P v)) on inner coarse DoFs for v vanishing on the
    boundary: nested P1 spaces (tests/test_solvers.cpp:231-270)."""
    mesh = FIXTURES[mesh_name]()
    L = 5
    dom = H.DistributedDomain(mesh, 2)
    ctl = H.Controller(dom)
    A = H.StencilOperator(dom, form, L - 1, L)
    v = H.ScalarFunction("v", dom, L - 1, L - 1)
    Ac_v = H.ScalarFunction("Acv", dom, L - 1, L - 1)
    Pv = H.ScalarFunction("Pv", dom, L, L)
    APv = H.ScalarFunction("APv", dom, L, L)
    RAPv = H.ScalarFunction("RAPv", dom, L - 1, L - 1)
    vv = keyed_uniform(mesh, L - 1, seed=7)
    vv[v.flags(L - 1) != H.INNER] = 0.0
    v.upload(L - 1, vv)
    H.apply(A, ctl, v, Ac_v, L - 1, H.INNER)
    H.prolongate(ctl, v, Pv, L - 1)
    H.apply(A, ctl, Pv, APv, L, H.INNER)
    H.restrict_to_coarse(ctl, APv, RAPv, L - 1)
    inner = v.flags(L - 1) == H.INNER
    want = Ac_v.download(L - 1)[inner]
    got = RAPv.download(L - 1)[inner]
    assert np.max(np.abs(got - want)) <= 1e-12 * max(1.0, np.max(np.abs(want)))


def energy(A, ctl, e, tmp, L):
    H.apply(A, ctl, e, tmp, L)
    return H.dot(e, tmp, L)


@pytest.mark.parametrize("mesh_name", ["square", "ring8", "channel21"])
@pytest.mark.parametrize("smoother", ["gs", "jacobi", "colored_gs"])
def test_smoothers_decrease_the_energy_norm(mesh_name, smoother):
    """With b = 0 every sweep shrinks ||e||_A (tests/test_operators.cpp:312-351)."""
    mesh = FIXTURES[mesh_name]()
    L = 5
    dom = H.DistributedDomain(mesh, 2)
    ctl = H.Controller(dom)
    A = H.StencilOperator(dom, H.LAPLACE, L, L)
    b = H.ScalarFunction("b", dom, L, L)
    e = H.ScalarFunction("e", dom, L, L)
    tmp = H.ScalarFunction("t", dom, L, L)
    ev = keyed_uniform(mesh, L, seed=8)
    ev[e.flags(L) != H.INNER] = 0.0
    e.upload(L, ev)
    last = energy(A, ctl, e, tmp, L)
    for _ in range(4):
        if smoother == "gs":
            H.smooth_gs(A, ctl, b, e, L)
        elif smoother == "colored_gs":
            H.smooth_colored_gs(A, ctl, b, e, L)
        else:
            H.smooth_jacobi(A, ctl, b, e, 2.0 / 3.0, L)
        now = energy(A, ctl, e, tmp, L)
        assert now < last, (smoother, now, last)
        last = now


@pytest.mark.parametrize("smoother", ["gs", "jacobi", "colored_gs"])
def test_zero_is_a_fixed_point_of_the_cycle(smoother):
    """rhs = 0, x = 0 stays exactly 0 (tests/test_solvers.cpp:394-406)."""
    mesh = FIXTURES["square"]()
    L = 5
    dom = H.DistributedDomain(mesh, 3)
    ctl = H.Controller(dom)
    rhs = H.ScalarFunction("rhs", dom, 1, L)
    x = H.ScalarFunction("x", dom, 1, L)
    mg = H.GridHierarchy(dom, ctl, H.LAPLACE, 1, L, smoother=smoother)
    for _ in range(3):
        mg.vcycle(rhs, x, L)
    assert np.all(x.download(L) == 0.0)


@pytest.mark.parametrize("smoother", ["jacobi", "gs"])
def test_mass_form_vcycle_converges_and_is_partition_invariant(smoother):
    """GridHierarchy with the MASS form (the reference's Form::MASS): the
    cycle converges, and its history and iterate are bitwise identical for 1
    and 3 ranks (the dot fold and the exchange are partition invariant)."""
    mesh = FIXTURES["ring8"]()
    L = 5
    out = []
    for ranks in (1, 3):
        dom = H.DistributedDomain(mesh, ranks)
        ctl = H.Controller(dom)
        rhs = H.ScalarFunction("rhs", dom, 1, L)
        x = H.ScalarFunction("x", dom, 1, L)
        b = keyed_uniform(mesh, L, seed=9)
        b[rhs.flags(L) != H.INNER] = 0.0
        rhs.upload(L, b)
        mg = H.GridHierarchy(dom, ctl, H.MASS, 1, L, smoother=smoother)
        rep = mg.solve(rhs, x, L, 0.0, 6)
        out.append((rep.residuals, x.download(L)))
    res = np.array(out[0][0])
    assert res[-1] / res[0] < 1e-4, res
    assert out[0][0] == out[1][0]
    assert np.array_equal(out[0][1], out[1][1])

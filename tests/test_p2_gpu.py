"""GPU parity of P2 (the reference's four-group quadratic kind,
src/operators.cpp:22-263 with FunctionKind::P2) through the C ABI against the
reference library itself (oracle/_ref), on the same inputs.

Bar: bitwise for apply (every form, masks), smooth_jacobi, smooth_gs and
diagonal -- the stencils are assembled in the reference's order and applied in
its term order; 1e-12 for dot (per-face partial order)."""
import numpy as np
import pytest

from oracle import ref as R
from paper_1805_10167_b200 import hytegrid as H
from tests.helpers import FIXTURES

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not R.available(), reason="oracle/_ref not built")]

MIXED_BC = {1: H.NEUMANN}


class P2Rig:
    def __init__(self, mesh, ranks, lmin, lmax, nfuncs=3, bc=None, form=H.LAPLACE):
        self.mesh, self.lmin, self.lmax = mesh, lmin, lmax
        self.dom = H.DistributedDomain(mesh, ranks)
        self.ctl = H.Controller(self.dom)
        self.f = [H.ScalarFunction(f"f{i}", self.dom, lmin, lmax, bc, kind=H.P2) for i in range(nfuncs)]
        self.A = H.StencilOperator(self.dom, form, lmin, lmax, bc, kind=H.P2)
        self.ref = R.RefSession(mesh, ranks, lmin, lmax, nfuncs, bc, kind=1)
        if form != H.LAPLACE:
            self.ref.set_form(form)
        self.rng = np.random.default_rng(17)

    def rand(self, i, level):
        v = self.rng.uniform(-1.0, 1.0, self.ref.owned(level))
        self.f[i].upload(level, v)
        self.ref.set(i, level, v)
        return v

    def check(self, i, level, what):
        mine, ref = self.f[i].download(level), self.ref.get(i, level)
        if not np.array_equal(mine.view(np.uint64), ref.view(np.uint64)):
            bad = np.flatnonzero(mine != ref)
            pytest.fail(f"{what}: {bad.size}/{mine.size} differ, first {bad[:6]}: {mine[bad[:6]]} vs {ref[bad[:6]]}")


CASES = [(m, r) for m in FIXTURES for r in (1, 2, 3)]


@pytest.mark.parametrize("mesh_name", list(FIXTURES))
def test_p2_counts_and_roundtrip(mesh_name):
    mesh = FIXTURES[mesh_name]()
    for ranks in (1, 3):
        for level in (0, 1, 3):
            rig = P2Rig(mesh, ranks, level, level, 1)
            n = rig.ref.owned(level)
            assert rig.dom.owned_count(level + 1)[0] == n   # P2 at L == P1 at L+1 (tests/test_functions.cpp:50)
            v = rig.rand(0, level)
            assert np.array_equal(rig.f[0].download(level), v)


@pytest.mark.parametrize("mesh_name,ranks", CASES)
@pytest.mark.parametrize("bc", [None, MIXED_BC], ids=["dirichlet", "mixed"])
def test_p2_apply_bitwise(mesh_name, ranks, bc):
    mesh = FIXTURES[mesh_name]()
    for level in range(0, 5):
        rig = P2Rig(mesh, ranks, level, level, 2, bc)
        rig.rand(0, level)
        rig.rand(1, level)  # masked rows must stay untouched
        for mask in (H.ALL_DOF_FLAGS, H.DIRICHLET, H.SMOOTH_MASK):
            H.apply(rig.A, rig.ctl, rig.f[0], rig.f[1], level, mask)
            rig.ref.apply(0, 1, level, mask)
            rig.check(1, level, f"P2 apply L{level} mask {mask}")


@pytest.mark.parametrize("form", [H.MASS, H.DIV_X, H.DIV_Y, H.GRAD_X, H.GRAD_Y, H.PSPG])
@pytest.mark.parametrize("mesh_name,ranks", [("square", 2), ("ring8", 3), ("channel21", 1)])
def test_p2_forms_apply_bitwise(form, mesh_name, ranks):
    mesh = FIXTURES[mesh_name]()
    for level in (1, 3):
        rig = P2Rig(mesh, ranks, level, level, 2, MIXED_BC, form=form)
        rig.rand(0, level)
        rig.rand(1, level)
        H.apply(rig.A, rig.ctl, rig.f[0], rig.f[1], level, H.ALL_DOF_FLAGS)
        rig.ref.apply(0, 1, level, H.ALL_DOF_FLAGS)
        rig.check(1, level, f"P2 form {form} L{level}")


@pytest.mark.parametrize("mesh_name,ranks", CASES)
def test_p2_smoothers_bitwise(mesh_name, ranks):
    mesh = FIXTURES[mesh_name]()
    for level in range(0, 5):
        for bc in (None, MIXED_BC):
            rig = P2Rig(mesh, ranks, level, level, 2, bc)
            rig.rand(0, level)  # rhs
            rig.rand(1, level)  # x
            for sweep in range(2):
                H.smooth_jacobi(rig.A, rig.ctl, rig.f[0], rig.f[1], 0.7, level)
                rig.ref.jacobi(0, 1, 0.7, level)
                rig.check(1, level, f"P2 Jacobi L{level} sweep {sweep}")
            for sweep in range(2):
                H.smooth_gs(rig.A, rig.ctl, rig.f[0], rig.f[1], level)
                rig.ref.gs(0, 1, level)
                rig.check(1, level, f"P2 GS L{level} sweep {sweep}")


@pytest.mark.parametrize("mesh_name,ranks", [("square", 1), ("ring8", 2), ("channel21", 3)])
def test_p2_diagonal_blas_dot(mesh_name, ranks):
    mesh = FIXTURES[mesh_name]()
    for level in (0, 2, 4):
        for form in (0, 1):
            rig = P2Rig(mesh, ranks, level, level, 3, MIXED_BC, form=form)
            H.diagonal(rig.A, rig.f[2], level)
            rig.ref.diagonal(form, 2, level)
            rig.check(2, level, f"P2 diagonal form {form} L{level}")
        a, b = rig.rand(0, level), rig.rand(1, level)
        H.assign(0.5, rig.f[0], -2.0, rig.f[1], rig.f[2], level, H.SMOOTH_MASK)
        rig.ref.assign(0.5, 0, -2.0, 1, 2, level, H.SMOOTH_MASK)
        rig.check(2, level, "P2 assign")
        H.add_scaled(rig.f[2], 3.0, rig.f[0], level, H.ALL_DOF_FLAGS)
        rig.ref.add_scaled(2, 3.0, 0, level, H.ALL_DOF_FLAGS)
        rig.check(2, level, "P2 add_scaled")
        d, dr = H.dot(rig.f[0], rig.f[1], level), rig.ref.dot(0, 1, level)
        assert abs(d - dr) <= 1e-12 * max(abs(dr), 1.0)
        assert H.dot(rig.f[0], rig.f[1], level) == pytest.approx(float(np.dot(a, b)), rel=1e-12, abs=1e-12)


def test_p2_exact_solution_is_a_gs_fixed_point():
    """tests/test_operators.cpp:287-310 with P2: x = A^-1 b on the interior is a
    fixed point of smooth_gs (checked against the reference's own sweep)"""
    mesh = FIXTURES["square"]()
    level = 3
    rig = P2Rig(mesh, 2, level, level, 2)
    rig.rand(1, level)
    H.apply(rig.A, rig.ctl, rig.f[1], rig.f[0], level, H.ALL_DOF_FLAGS)  # b = A x (DIRICHLET rows b = x)
    rig.ref.apply(1, 0, level, H.ALL_DOF_FLAGS)
    x0 = rig.f[1].download(level)
    H.smooth_gs(rig.A, rig.ctl, rig.f[0], rig.f[1], level)
    assert np.max(np.abs(rig.f[1].download(level) - x0)) <= 1e-12


def test_p2_kind_errors():
    mesh = FIXTURES["square"]()
    dom = H.DistributedDomain(mesh, 1)
    ctl = H.Controller(dom)
    A2 = H.StencilOperator(dom, H.LAPLACE, 2, 2, kind=H.P2)
    f1 = H.ScalarFunction("p1", dom, 1, 2)
    f2 = H.ScalarFunction("p2", dom, 1, 2, kind=H.P2)
    g2 = H.ScalarFunction("g2", dom, 1, 2, kind=H.P2)
    with pytest.raises(H.InvalidArgument, match="kind"):
        H.apply(A2, ctl, f1, g2, 2)
    with pytest.raises(H.InvalidArgument, match="different function kinds"):
        H.assign(1.0, f1, 1.0, f2, g2, 2)
    with pytest.raises(H.InvalidArgument, match="defined for P1"):
        H.prolongate(ctl, f2, g2, 1)
    with pytest.raises(H.InvalidArgument, match="P1"):
        H.residual(A2, ctl, f2, g2, H.ScalarFunction("r", dom, 1, 2, kind=H.P2), 2)


@pytest.mark.parametrize("mesh_name", list(FIXTURES))
def test_p2_coordinates_and_interpolate(mesh_name):
    """P2 DoF coordinates (for_each_owned_coord with P2, src/layout.cpp:239-282)
    are bitwise the reference's, in its P2 order; interpolate evaluates there"""
    mesh = FIXTURES[mesh_name]()
    for ranks in (1, 2):
        for level in (0, 2, 3):
            rig = P2Rig(mesh, ranks, level, level, 1)
            xy = rig.dom.coords(level, kind=H.P2)
            assert np.array_equal(xy, rig.ref.coords(level))
            H.interpolate(rig.f[0], lambda x, y: x * x - 3.0 * y, level, H.SMOOTH_MASK)
            fl = rig.ref.flags(0, level)
            want = np.where(fl & H.SMOOTH_MASK, xy[:, 0] * xy[:, 0] - 3.0 * xy[:, 1], 0.0)
            assert np.array_equal(rig.f[0].download(level), want)

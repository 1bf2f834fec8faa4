"""The two-sweep Jacobi pass (temporal blocking, ST_JACOBI2): bitwise two
smooth_jacobi sweeps -- on the face interiors two or more away from every
border (formed from x1 in registers), the layers next to the borders and the
edges/vertices -- over meshes, ranks, boundary conditions and levels that
exercise one and several column blocks and bands; and V-cycles with the pass
(graph-replayed, arenas restored) bitwise the cycles without it."""
import os

import numpy as np
import pytest

from oracle import ref as R
from paper_1805_10167_b200 import hytegrid as H
from tests.helpers import FIXTURES, keyed_uniform

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _pass_on():
    """the pass is off by default (slower than two sweeps on B200): test it on"""
    prev = H.tuning("jacobi2_min_n", 16)
    yield
    H.tuning("jacobi2_min_n", prev)


def two_ways(mesh, ranks, level, bc, omega=0.7):
    out = []
    for fused in (True, False):
        dom = H.DistributedDomain(mesh, ranks)
        ctl = H.Controller(dom)
        A = H.StencilOperator(dom, H.LAPLACE, level, level, bc)
        x, b = H.ScalarFunction("x", dom, level, level, bc), H.ScalarFunction("b", dom, level, level, bc)
        x.upload(level, keyed_uniform(mesh, level, 21))
        b.upload(level, keyed_uniform(mesh, level, 22))
        for _ in range(2):
            if fused:
                H.smooth_jacobi2(A, ctl, b, x, omega, level)
            else:
                H.smooth_jacobi(A, ctl, b, x, omega, level)
                H.smooth_jacobi(A, ctl, b, x, omega, level)
        out.append(x.download(level))
    return out


@pytest.mark.parametrize("mesh_name", list(FIXTURES))
@pytest.mark.parametrize("ranks", [1, 3])
@pytest.mark.parametrize("bc", [None, {1: H.NEUMANN}], ids=["dirichlet", "mixed"])
def test_two_sweep_pass_bitwise(mesh_name, ranks, bc):
    mesh = FIXTURES[mesh_name]()
    for level in (6, 7, 9):
        fused, plain = two_ways(mesh, ranks, level, bc)
        assert np.array_equal(fused.view(np.uint64), plain.view(np.uint64)), (mesh_name, ranks, level)


def test_two_sweep_pass_vs_reference():
    """and against the reference library itself: two of its smooth_jacobi calls"""
    if not R.available():
        pytest.skip("oracle/_ref not built")
    mesh = H.meshgen.annulus(8, 2, 1.0, 2.0)
    level = 7
    fused, _ = two_ways(mesh, 2, level, None)
    ref = R.RefSession(mesh, 2, level, level, 2)
    ref.set(0, level, keyed_uniform(mesh, level, 21))
    ref.set(1, level, keyed_uniform(mesh, level, 22))
    for _ in range(4):
        ref.jacobi(1, 0, 0.7, level)
    assert np.array_equal(fused, ref.get(0, level))


@pytest.mark.parametrize("ranks", [1, 2])
@pytest.mark.parametrize("nu", [(2, 2), (2, 3)])
def test_vcycles_with_the_pass_bitwise(ranks, nu):
    mesh = H.meshgen.channel(4, 4)
    L = 8
    res = []
    for temporal in (True, False):
        dom = H.DistributedDomain(mesh, ranks)
        ctl = H.Controller(dom)
        mg = H.GridHierarchy(dom, ctl, H.LAPLACE, 0, L, smoother="jacobi")
        assert mg.use_temporal(temporal) == temporal
        rhs, x = H.ScalarFunction("b", dom, 0, L), H.ScalarFunction("x", dom, 0, L)
        rhs.upload(L, keyed_uniform(mesh, L, 5))
        rep = mg.solve(rhs, x, L, 0.0, 6, *nu)
        res.append((np.array(rep.residuals), x.download(L), mg.use_graphs()))
    assert np.array_equal(res[0][0], res[1][0]) and np.array_equal(res[0][1], res[1][1])
    if sum(nu) % 2 == 0:
        assert res[0][2] > 0  # the cycles with the pass replayed from CUDA graphs

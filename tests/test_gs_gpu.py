"""GPU parity of the hybrid Gauss-Seidel smoother (reference smooth_gs,
src/operators.cpp:423-482) and of the reference's own GridHierarchy (which
smooths with it, src/solvers.cpp:406-428): bitwise per sweep, 1e-8 per cycle
for residual histories."""
import numpy as np
import pytest

from oracle import ref as R
from paper_1805_10167_b200 import hytegrid as H
from tests.helpers import FIXTURES, keyed_uniform, probe

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not R.available(), reason="oracle/_ref not built")]


def _rig(mesh, ranks, lmin, lmax, bc=None):
    dom = H.DistributedDomain(mesh, ranks)
    A = H.StencilOperator(dom, H.LAPLACE, lmin, lmax, bc)
    f = [H.ScalarFunction(f"f{i}", dom, lmin, lmax, bc) for i in range(2)]
    ref = R.RefSession(mesh, ranks, lmin, lmax, 2, bc)
    return dom, H.Controller(dom), A, f, ref


@pytest.mark.parametrize("mesh_name", sorted(FIXTURES))
@pytest.mark.parametrize("ranks", [1, 2, 3])
def test_gs_sweeps_bitwise(mesh_name, ranks):
    mesh = FIXTURES[mesh_name]()
    for level in (1, 2, 3, 5, 6):
        bc = {1: H.NEUMANN} if ranks == 2 else None
        dom, ctl, A, f, ref = _rig(mesh, ranks, level, level, bc)
        for i, seed in ((0, 41), (1, 42)):
            v = keyed_uniform(mesh, level, seed)
            f[i].upload(level, v)
            ref.set(i, level, v)
        for sweep in range(3):
            H.smooth_gs(A, ctl, f[0], f[1], level)
            ref.gs(0, 1, level)
            mine, want = f[1].download(level), ref.get(1, level)
            assert np.array_equal(mine, want), (mesh_name, ranks, level, sweep,
                                                np.flatnonzero(mine != want)[:5])


@pytest.mark.slow
def test_gs_bitwise_cfg2_mesh_level8():
    """512 faces at level 8: 64 tiles per face, many tile wavefronts in flight."""
    mesh = H.meshgen.channel(16, 16)
    L = 8
    dom, ctl, A, f, ref = _rig(mesh, 1, L, L)
    for i, seed in ((0, 1), (1, 2)):
        v = keyed_uniform(mesh, L, seed)
        f[i].upload(L, v)
        ref.set(i, L, v)
    for _ in range(2):
        H.smooth_gs(A, ctl, f[0], f[1], L)
        ref.gs(0, 1, L)
    assert np.array_equal(f[1].download(L), ref.get(1, L))


def test_gs_annulus_perturbed_bitwise():
    """Per-face affine stencils with all six couplings non-zero (config 3 mesh family)."""
    mesh = H.meshgen.perturb(H.meshgen.annulus(16, 4, 1.0, 2.0), 0.1, 2)
    L = 6
    dom, ctl, A, f, ref = _rig(mesh, 2, L, L)
    for i, seed in ((0, 3), (1, 4)):
        v = keyed_uniform(mesh, L, seed)
        f[i].upload(L, v)
        ref.set(i, L, v)
    for _ in range(2):
        H.smooth_gs(A, ctl, f[0], f[1], L)
        ref.gs(0, 1, L)
    assert np.array_equal(f[1].download(L), ref.get(1, L))


@pytest.mark.parametrize("mesh_name,ranks,lmax", [("square", 2, 5), ("square_rev", 3, 4), ("ring8", 2, 5),
                                                  ("channel21", 1, 5)])
def test_gridhierarchy_gs_matches_reference(mesh_name, ranks, lmax):
    """Device GridHierarchy with the reference's smoother vs the reference's
    own GridHierarchy::solve (tests/test_solvers.cpp:431-462 setup)."""
    mesh = FIXTURES[mesh_name]()
    dom = H.DistributedDomain(mesh, ranks)
    ctl = H.Controller(dom)
    mg = H.GridHierarchy(dom, ctl, H.LAPLACE, 1, lmax, smoother="gs", coarse_tol=1e-12)
    rhs = H.ScalarFunction("rhs", dom, 1, lmax)
    x = H.ScalarFunction("x", dom, 1, lmax)
    ref = R.RefSession(mesh, ranks, 1, lmax, 2)
    xy = dom.coords(lmax)
    x0 = probe(xy[:, 0], xy[:, 1])
    flags = x.flags(lmax)
    x0[flags == H.DIRICHLET] = 0.0
    x.upload(lmax, x0)
    ref.set(1, lmax, x0)
    rep = mg.solve(rhs, x, lmax, 0.0, 10)
    ref_hist = ref.gridhierarchy_solve(0, 1, lmax, 0.0, 10)
    mine = np.array(rep.residuals)
    assert mine.shape == ref_hist.shape
    assert np.max(np.abs(mine - ref_hist) / ref_hist) <= 1e-8, (mine, ref_hist)
    assert mine[10] < mine[0]


@pytest.mark.parametrize("ranks", [2, 4])
def test_gs_partition_invariance(ranks):
    # reference tests/test_operators.cpp:353-370
    mesh = H.meshgen.square_ring8()
    out = []
    for rk in (1, ranks):
        dom = H.DistributedDomain(mesh, rk)
        A = H.StencilOperator(dom, H.LAPLACE, 4, 4)
        x = H.ScalarFunction("x", dom, 4, 4)
        rhs = H.ScalarFunction("rhs", dom, 4, 4)
        H.interpolate(x, probe, 4)
        for _ in range(10):
            H.smooth_gs(A, H.Controller(dom), rhs, x, 4)
        out.append(x.download(4))
    assert np.array_equal(out[0], out[1])

"""GPU checks of the BASELINE configurations beyond config 1/2:

config 3 -- perturbed annulus, per-face affine stencils, V(3,3) with coloured
Gauss-Seidel (the reference has no coloured GS; the checker is the C
restatement oracle/hyteg_oracle.c og_cgs, whose plain GS branch is pinned
bitwise to the reference). Reduced sizes against the oracle, bitwise per sweep
and 1e-8 per cycle; the full size (level 9, 1.07 G DoFs) through convergence
properties."""
import numpy as np
import pytest

from oracle import restatement as O
from paper_1805_10167_b200 import hytegrid as H
from tests.helpers import FIXTURES, keyed_uniform

pytestmark = pytest.mark.gpu


def cfg3_mesh(segments=128, layers=32):
    # interior coarse vertices moved by U[-0.1, 0.1] x shortest incident edge (seed 2)
    return H.meshgen.perturb(H.meshgen.annulus(segments, layers, 1.0, 2.0), 0.1, 2)


@pytest.mark.parametrize("mesh_name", ["square", "square_rev", "ring8", "channel21", "annulus"])
@pytest.mark.parametrize("ranks", [1, 3])
def test_colored_gs_bitwise_vs_restatement(mesh_name, ranks):
    mesh = cfg3_mesh(16, 4) if mesh_name == "annulus" else FIXTURES[mesh_name]()
    for level in (1, 2, 4, 6):
        dom = H.DistributedDomain(mesh, ranks)
        ctl = H.Controller(dom)
        A = H.StencilOperator(dom, H.LAPLACE, level, level)
        rhs, x = H.ScalarFunction("rhs", dom, level, level), H.ScalarFunction("x", dom, level, level)
        o = O.Session(mesh, level, level, 2)
        for f, i, seed in ((rhs, 0, 51), (x, 1, 52)):
            v = keyed_uniform(mesh, level, seed)
            f.upload(level, v)
            o.set(i, level, v)
        for sweep in range(3):
            H.smooth_colored_gs(A, ctl, rhs, x, level)
            o.cgs(0, 1, level)
            assert np.array_equal(x.download(level), o.get(1, level)), (mesh_name, ranks, level, sweep)


def test_cfg3_reduced_vcycle_history():
    """Config 3 shape at reduced size: perturbed annulus(32, 8) levels 5 -> 0,
    V(3,3) coloured GS, rhs U[-1,1] (seed 2) on INNER, x0 = 0, 5 cycles."""
    mesh = cfg3_mesh(32, 8)
    L = 5
    dom = H.DistributedDomain(mesh, 2)
    ctl = H.Controller(dom)
    rhs = H.ScalarFunction("rhs", dom, 0, L)
    x = H.ScalarFunction("x", dom, 0, L)
    b = keyed_uniform(mesh, L, seed=2)
    b[rhs.flags(L) != H.INNER] = 0.0
    rhs.upload(L, b)
    mg = H.GridHierarchy(dom, ctl, H.LAPLACE, 0, L, smoother="colored_gs", coarse_tol=1e-12)
    rep = mg.solve(rhs, x, L, 0.0, 5, 3, 3)
    o = O.Session(mesh, 0, L, 7)
    o.set(0, L, b)
    ref = o.vcycle(0, 1, L, 2, 3, 3, 1.0, 1e-12, 5)
    mine = np.array(rep.residuals)
    assert np.max(np.abs(mine - ref) / ref) <= 1e-8, (mine, ref)
    assert mine[-1] / mine[0] < 0.05


@pytest.mark.slow
def test_cfg3_full_size():
    """Config 3 at full size: annulus 128 x 32 (8192 faces), level 9, V(3,3)
    coloured GS, 5 cycles: residual falls every cycle."""
    mesh = cfg3_mesh()
    L = 9
    dom = H.DistributedDomain(mesh, 1)
    assert dom.owned_count(L)[0] == 1_073_807_360
    ctl = H.Controller(dom)
    rhs = H.ScalarFunction("rhs", dom, 0, L)
    x = H.ScalarFunction("x", dom, 0, L)
    H.interpolate_random(rhs, L, seed=2, flag_mask=H.INNER)
    mg = H.GridHierarchy(dom, ctl, H.LAPLACE, 0, L, smoother="colored_gs", coarse_tol=1e-12)
    rep = mg.solve(rhs, x, L, 0.0, 5, 3, 3)
    res = np.array(rep.residuals)
    assert np.all(res[1:] < res[:-1]), res
    assert res[-1] / res[0] < 1e-2, res

"""prolongate(add) fused into the first coloured post-sweep (k_cgs_cols<PRO>,
hyb_prolongate_add_cgs): bitwise the two operations in sequence.

Checked against the C restatement (og_prolongate into a scratch function,
add_scaled on the smooth mask, og_cgs) on faces of n = 256 (in place) and 512 /
1024 (256-column blocks, out of place), 1 and 3 ranks; against the product's
own unfused calls under mixed boundary conditions; and through coloured-GS
V-cycles with the fusion on and off."""
import numpy as np
import pytest

from oracle import restatement as O
from paper_1805_10167_b200 import hytegrid as H
from tests.helpers import FIXTURES, keyed_uniform

pytestmark = pytest.mark.gpu

SMOOTH = H.INNER | H.NEUMANN


@pytest.fixture
def fused_on():
    prev = H.tuning("cgs_prolong_fused", 1)
    yield
    H.tuning("cgs_prolong_fused", prev)


def cfg3_mesh(segments, layers):
    return H.meshgen.perturb(H.meshgen.annulus(segments, layers, 1.0, 2.0), 0.1, 2)


@pytest.mark.parametrize("mesh_name,level", [("square", 8), ("square", 9), ("square", 10), ("annulus", 8),
                                             ("annulus", 9)])
@pytest.mark.parametrize("ranks", [1, 3])
def test_fused_vs_restatement(fused_on, mesh_name, level, ranks):
    mesh = cfg3_mesh(4, 2) if mesh_name == "annulus" else FIXTURES[mesh_name]()
    lc = level - 1
    dom = H.DistributedDomain(mesh, ranks)
    ctl = H.Controller(dom)
    A = H.StencilOperator(dom, H.LAPLACE, lc, level)
    rhs, x = H.ScalarFunction("rhs", dom, lc, level), H.ScalarFunction("x", dom, lc, level)
    e = H.ScalarFunction("e", dom, lc, level)
    o = O.Session(mesh, lc, level, 4)
    for f, i, seed, L in ((rhs, 0, 91, level), (x, 1, 92, level), (e, 2, 93, lc)):
        v = keyed_uniform(mesh, L, seed)
        f.upload(L, v)
        o.set(i, L, v)
    o.set(3, level, np.zeros_like(o.get(3, level)))
    H.prolongate_add_colored_gs(A, ctl, e, rhs, x, lc)
    o.prolongate(2, 3, lc, SMOOTH)
    o.add_scaled(1, 1.0, 3, level, SMOOTH)
    o.cgs(0, 1, level)
    assert np.array_equal(x.download(level), o.get(1, level)), (mesh_name, level, ranks)


@pytest.mark.parametrize("level", [8, 9])
def test_fused_mixed_bc_vs_unfused(fused_on, level):
    mesh = FIXTURES["channel21"]()
    bc = {1: H.DIRICHLET, 2: H.DIRICHLET, 3: H.NEUMANN}
    lc = level - 1
    out = []
    for fused in (True, False):
        dom = H.DistributedDomain(mesh, 2)
        ctl = H.Controller(dom)
        A = H.StencilOperator(dom, H.LAPLACE, lc, level, bc)
        rhs = H.ScalarFunction("rhs", dom, lc, level, bc)
        x = H.ScalarFunction("x", dom, lc, level, bc)
        e = H.ScalarFunction("e", dom, lc, level, bc)
        rhs.upload(level, keyed_uniform(mesh, level, 94))
        x.upload(level, keyed_uniform(mesh, level, 95))
        e.upload(lc, keyed_uniform(mesh, lc, 96))
        if fused:
            H.prolongate_add_colored_gs(A, ctl, e, rhs, x, lc)
        else:
            H.prolongate_add(ctl, e, x, lc, SMOOTH)
            H.smooth_colored_gs(A, ctl, rhs, x, level)
        out.append(x.download(level))
    assert np.array_equal(out[0], out[1])


@pytest.mark.parametrize("nu", [(3, 3), (2, 1), (1, 2)])
def test_cycles_fused_vs_unfused(nu):
    """Coloured-GS V-cycles L9 -> 0 with the fusion on and off: the same iterates bitwise over
    four cycles (eager, warm, captured, replayed)."""
    mesh = cfg3_mesh(4, 2)
    L = 9
    res = []
    for on in (1, 0):
        prev = H.tuning("cgs_prolong_fused", on)
        try:
            dom = H.DistributedDomain(mesh, 1)
            ctl = H.Controller(dom)
            mg = H.GridHierarchy(dom, ctl, H.LAPLACE, 0, L, smoother="colored_gs", coarse_tol=1e-12)
            rhs, x = H.ScalarFunction("rhs", dom, 0, L), H.ScalarFunction("x", dom, 0, L)
            H.interpolate_random(rhs, L, seed=6, flag_mask=H.INNER)
            it = []
            for _ in range(4):
                mg.vcycle(rhs, x, L, *nu)
                it.append(x.download(L))
            res.append(it)
        finally:
            H.tuning("cgs_prolong_fused", prev)
    for a, b in zip(*res):
        assert np.array_equal(a, b), nu

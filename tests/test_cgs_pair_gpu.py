"""Two coloured sweeps in one face pass (k_cgs_pair, hyb_smooth_cgs_n).

The pass must be bitwise two smooth_cgs calls: the faces' sweep 2 reads the
boundary ghosts after the sweep-1 refresh, the edges' sweep 2 reads the faces'
sweep-1 layer. Checked against the C restatement (og_cgs, one sweep at a time)
on face sizes 256 (in place) and 512 (two column blocks, out of place), with 1
rank (pairs used) and 3 ranks (the fallback: singles); against the product's
own single sweeps under mixed boundary conditions; and through V(3,3) / V(3,1)
coloured-GS cycles (graph replay, and the eager fallback for a cycle that
leaves an arena swapped)."""
import numpy as np
import pytest

from oracle import restatement as O
from paper_1805_10167_b200 import hytegrid as H
from tests.helpers import FIXTURES, keyed_uniform

pytestmark = pytest.mark.gpu


def cfg3_mesh(segments, layers):
    return H.meshgen.perturb(H.meshgen.annulus(segments, layers, 1.0, 2.0), 0.1, 2)


@pytest.fixture
def pairs_on():
    prev = H.tuning("cgs_pair_min_n", 256)
    yield
    H.tuning("cgs_pair_min_n", prev)


@pytest.mark.parametrize("mesh_name", ["square", "annulus"])
@pytest.mark.parametrize("ranks", [1, 3])
@pytest.mark.parametrize("level", [8, 9])
def test_pair_bitwise_vs_restatement(pairs_on, mesh_name, ranks, level):
    mesh = cfg3_mesh(4, 2) if mesh_name == "annulus" else FIXTURES[mesh_name]()
    dom = H.DistributedDomain(mesh, ranks)
    ctl = H.Controller(dom)
    A = H.StencilOperator(dom, H.LAPLACE, level, level)
    rhs, x = H.ScalarFunction("rhs", dom, level, level), H.ScalarFunction("x", dom, level, level)
    o = O.Session(mesh, level, level, 2)
    for f, i, seed in ((rhs, 0, 71), (x, 1, 72)):
        v = keyed_uniform(mesh, level, seed)
        f.upload(level, v)
        o.set(i, level, v)
    done = 0
    for count in (2, 3, 4):  # a pair; a pair + a single; two pairs
        H.smooth_colored_gs(A, ctl, rhs, x, level, count=count)
        for _ in range(count):
            o.cgs(0, 1, level)
        done += count
        assert np.array_equal(x.download(level), o.get(1, level)), (mesh_name, ranks, level, done)


@pytest.mark.parametrize("level", [8, 9])
def test_pair_mixed_bc_vs_singles(pairs_on, level):
    mesh = FIXTURES["channel21"]()
    bc = {1: H.DIRICHLET, 2: H.DIRICHLET, 3: H.NEUMANN}
    out = []
    for count in (1, 4):
        dom = H.DistributedDomain(mesh, 1)
        ctl = H.Controller(dom)
        A = H.StencilOperator(dom, H.LAPLACE, level, level, bc)
        rhs = H.ScalarFunction("rhs", dom, level, level, bc)
        x = H.ScalarFunction("x", dom, level, level, bc)
        rhs.upload(level, keyed_uniform(mesh, level, 81))
        x.upload(level, keyed_uniform(mesh, level, 82))
        if count == 1:
            for _ in range(4):
                H.smooth_colored_gs(A, ctl, rhs, x, level)
        else:
            H.smooth_colored_gs(A, ctl, rhs, x, level, count=4)
        out.append(x.download(level))
    assert np.array_equal(out[0], out[1])


@pytest.mark.parametrize("nu", [(3, 3), (3, 1), (2, 2)])
def test_cgs_cycles_pairs_vs_singles(nu):
    """V-cycles with the pair pass (levels 8, 9) and without: the same iterates bitwise, over
    four cycles (eager, warm, captured, replayed; V(3,1) stays eager after its capture)."""
    mesh = cfg3_mesh(4, 2)
    L = 9
    res = []
    for min_n in (256, 1 << 30):
        prev = H.tuning("cgs_pair_min_n", min_n)
        try:
            dom = H.DistributedDomain(mesh, 1)
            ctl = H.Controller(dom)
            mg = H.GridHierarchy(dom, ctl, H.LAPLACE, 0, L, smoother="colored_gs", coarse_tol=1e-12)
            rhs, x = H.ScalarFunction("rhs", dom, 0, L), H.ScalarFunction("x", dom, 0, L)
            H.interpolate_random(rhs, L, seed=5, flag_mask=H.INNER)
            it = []
            for _ in range(4):
                mg.vcycle(rhs, x, L, *nu)
                it.append(x.download(L))
            res.append(it)
        finally:
            H.tuning("cgs_pair_min_n", prev)
    for a, b in zip(*res):
        assert np.array_equal(a, b), nu

"""Communication/computation overlap (the paper's Algorithm 3): with ghosts
owned by other ranks, apply / residual / Jacobi run the interior primitives
while the exchange is in flight and the boundary ones after it. Checked on one
GPU with co-resident logical ranks (their ghosts travel through the same
pack / transfer / receive path as NCCL's): bitwise the unsplit launches, and
the reference's results through the parity tests that run with it on."""
import numpy as np
import pytest

from paper_1805_10167_b200 import hytegrid as H
from tests.helpers import FIXTURES, keyed_uniform

pytestmark = pytest.mark.gpu


def run(mesh, ranks, level, overlap, bc=None):
    dom = H.DistributedDomain(mesh, ranks)
    dom.overlap(overlap)
    ctl = H.Controller(dom)
    A = H.StencilOperator(dom, H.LAPLACE, level, level, bc)
    x, b, y, r = (H.ScalarFunction(n, dom, level, level, bc) for n in "xbyr")
    H.interpolate_random(x, level, 3, 0)
    H.interpolate_random(b, level, 3, 1)
    out = []
    H.apply(A, ctl, x, y, level)
    out.append(y.download(level))
    H.residual(A, ctl, b, x, r, level)
    out.append(r.download(level))
    for _ in range(3):
        H.smooth_jacobi(A, ctl, b, x, 0.7, level)
    out.append(x.download(level))
    return out, dom.overlap()


@pytest.mark.parametrize("mesh_name", list(FIXTURES))
@pytest.mark.parametrize("ranks", [2, 3])
def test_overlap_is_bitwise_the_unsplit_launch(mesh_name, ranks):
    mesh = FIXTURES[mesh_name]()
    for level in (2, 5):
        for bc in (None, {1: H.NEUMANN}):
            split, nsplit = run(mesh, ranks, level, True, bc)
            plain, nplain = run(mesh, ranks, level, False, bc)
            assert nsplit > 0 and nplain == 0
            for a, b in zip(split, plain):
                assert np.array_equal(a.view(np.uint64), b.view(np.uint64))


def test_one_rank_has_nothing_to_overlap():
    _, n = run(FIXTURES["square"](), 1, 4, True)
    assert n == 0


@pytest.mark.parametrize("ranks", [2, 4])
def test_overlapped_vcycles_graph_replayed(ranks):
    """V-cycles (CUDA-graph captured, the communication stream forks and joins
    inside the capture) with and without overlap: identical histories"""
    mesh = H.meshgen.channel(4, 4)
    hist = []
    for ov in (True, False):
        dom = H.DistributedDomain(mesh, ranks)
        dom.overlap(ov)
        ctl = H.Controller(dom)
        mg = H.GridHierarchy(dom, ctl, H.LAPLACE, 0, 6, smoother="jacobi")
        rhs, x = H.ScalarFunction("b", dom, 0, 6), H.ScalarFunction("x", dom, 0, 6)
        rhs.upload(6, keyed_uniform(mesh, 6, 4))
        rep = mg.solve(rhs, x, 6, 0.0, 6)
        hist.append((np.array(rep.residuals), x.download(6), mg.use_graphs()))
    assert np.array_equal(hist[0][0], hist[1][0])
    assert np.array_equal(hist[0][1], hist[1][1])
    assert hist[0][2] > 0  # graph replays happened with overlap on

"""Device interpolation of analytic expressions (hyb_interpolate_expr) against the same expressions
evaluated on the host at the reference's DoF coordinates (hyb_owned_coords, bitwise the reference's
for_each_owned_coord, src/layout.cpp:239-282)."""
import numpy as np
import pytest

from paper_1805_10167_b200 import hytegrid as H
from tests.helpers import FIXTURES

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("mesh_name", ["square", "ring8", "channel21"])
@pytest.mark.parametrize("ranks", [1, 3])
def test_poly2_bitwise_host_evaluation(mesh_name, ranks):
    mesh = FIXTURES[mesh_name]()
    p = [0.25, -1.5, 2.0, 0.75, -0.125, 3.0]
    for level in (0, 1, 3, 6):
        dom = H.DistributedDomain(mesh, ranks)
        f = H.ScalarFunction("f", dom, level, level)
        H.interpolate_expr(f, level, H.EXPR_POLY2, p)
        xy = dom.coords(level)
        x, y = xy[:, 0], xy[:, 1]
        want = ((((p[0] + p[1] * x) + p[2] * y) + p[3] * (x * x)) + p[4] * (x * y)) + p[5] * (y * y)
        assert np.array_equal(f.download(level), want), (mesh_name, ranks, level)


def test_sinsin_matches_host_and_masks():
    mesh = FIXTURES["square"]()
    L = 7
    dom = H.DistributedDomain(mesh, 1)
    f = H.ScalarFunction("f", dom, L, L)
    H.interpolate(f, -2.0, L)
    p = [1.0, np.pi, 0.0, np.pi, 0.0, 0.5]
    H.interpolate_expr(f, L, H.EXPR_SINSIN, p, flag_mask=H.INNER)
    xy = dom.coords(L)
    want = p[0] * np.sin(p[1] * xy[:, 0] + p[2]) * np.sin(p[3] * xy[:, 1] + p[4]) + p[5]
    got = f.download(L)
    inner = f.flags(L) == H.INNER
    assert np.all(got[~inner] == -2.0)  # DIRICHLET rows untouched by the INNER mask
    err = np.abs(got[inner] - want[inner])
    assert err.max() <= 4 * np.finfo(np.float64).eps * np.abs(want[inner]).max()  # libm vs CUDA sin


def test_expr_errors():
    dom = H.DistributedDomain(FIXTURES["square"](), 1)
    f = H.ScalarFunction("f", dom, 2, 2)
    with pytest.raises(ValueError):
        H.interpolate_expr(f, 2, 7, [1.0])
    with pytest.raises(ValueError):
        H.interpolate_expr(f, 2, H.EXPR_POLY2, np.zeros(9))
    with pytest.raises(IndexError):
        H.interpolate_expr(f, 5, H.EXPR_POLY2, [1.0])
